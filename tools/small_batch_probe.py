import os, sys, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import lora_inputs as li
from paper_2604_07173_b200 import binding as B
sys.path.insert(0, '/root/repo/tools')
import layout_table as LT

def prof_run(cfg, b, fake=None, y=1, small=None):
    if fake: os.environ["LORA_FAKE_WORLD"] = fake
    c = B.make_config([s.h_in for s in cfg.slots], [s.h_out for s in cfg.slots], [s.n_experts for s in cfg.slots],
                      cfg.rank, cfg.n_adapters, cfg.scale(), b.n_rows, 0, expert_parallel=bool(fake), pp_stages=y,
                      slot_layer=[0]*3)
    s = B.lora_server_create(c)
    if fake: del os.environ["LORA_FAKE_WORLD"]
    if small is not None: B.lora_server_set_small_seg_max(s, small)
    B.lora_server_fill_synthetic(s, cfg.seed)
    T = b.n_rows; dev = torch.device('cuda', 0)
    xs = {}
    for i, sl in enumerate(cfg.slots):
        if sl.xbuf not in xs:
            x = torch.empty((T, sl.h_in), dtype=torch.int16, device=dev)
            B.lora_synth_fill_rows(x, T, sl.h_in, cfg.seed, li.tag_of(li.KIND_X, sl.xbuf), li.shift_x(), 0)
            xs[sl.xbuf] = x
    ys = [torch.zeros((T, sl.h_out), dtype=torch.int16, device=dev) for sl in cfg.slots]
    ad = torch.from_numpy(b.adapter_ids).to(dev); ex = torch.from_numpy(b.expert_ids).to(dev)
    p = B.lora_plan_create(s, T)
    xl = [xs[sl.xbuf] for sl in cfg.slots]
    for it in range(3):
        B.lora_plan_build(s, p, ad, ex, T, 8); B.lora_apply_plan_multi(s, p, [0,1,2], xl, ys, B.LORA_BF16)
    torch.cuda.synchronize()
    st = B.lora_plan_stats(s, p)
    res = {}
    for conc in (True, False):
        B.lora_server_set_concurrent(s, conc)
        B.lora_profile_enable(s, 200)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for it in range(5):
            B.lora_plan_build(s, p, ad, ex, T, 8); B.lora_apply_plan_multi(s, p, [0,1,2], xl, ys, B.LORA_BF16)
        e1.record(); torch.cuda.synchronize()
        pr = B.lora_profile_read(s); B.lora_profile_enable(s, 0)
        res["conc" if conc else "serial"] = {"step_us": e0.elapsed_time(e1)/5*1e3, **{k: round(v[1]/5*1e3,1) for k, v in pr.items()}}
    B.lora_server_check(s); B.lora_plan_destroy(p); B.lora_server_destroy(s)
    return st, res

base = li.CONFIGS["mixtral_decode"]
for ntok in (64, 128, 512):
    cfg = li.with_tokens(base, ntok); b = li.make_batch(cfg)
    for small in (None, -1):
        print("full", ntok, "small", small, prof_run(cfg, b, None, 1, small), flush=True)
cfg = li.with_tokens(base, 128); b = li.make_batch(cfg)
for small in (None, -1):
    print("EP8 r0", prof_run(cfg, b, "8,0,1,0,1", 1, small), flush=True)
    print("EP4 r0", prof_run(cfg, b, "8,0,1,0,2", 2, small), flush=True)
