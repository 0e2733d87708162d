#!/usr/bin/env python
"""Table-BD analog (tab:time_breakdown_on_epx_ppy): LoRA
execution of one Mixtral layer under the four EP_x-PP_y layouts of an
8-GPU LoRA Server (EP1-PP8, EP2-PP4, EP4-PP2, EP8-PP1), decode batches of 128
and 256 tokens (top-2 -> 256 / 512 rows), 512 adapters, Zipf(1.2).

Compute (measured, one B200): for each rank of the group that owns layer 0
(x ranks), a fake-world store of exactly that rank's units (LORA_FAKE_WORLD=
8,rank,1,0,y: hybrid placement, owner = (l mod y) * x + e mod x) applies the
whole batch; the segmenter keeps only the rows that rank owns, so the timed
step is that rank's plan build + gate/up/down apply on its rows, CUDA graph
replay, median of 20.  The layout's LoRA time is the slowest rank of the group.

Exchange (modelled, printed beside it): each owner receives its rows' x from
the clients and returns their deltas (Table 1: peer volume b*k / max(p, x),
peer count max(p / x, 1), sync scope x); on one NVLink domain the push path
fuses both transfers into the kernels, so the step is modelled as
max(compute, exchange at 700 GB/s) -- no separate synchronisation term.

    python tools/layout_table.py > profiles/r2_layout_table.json
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import lora_inputs as li  # noqa: E402
from oracle import oracle as orc  # noqa: E402 (routing rule only: owner_of)

G = 8


def rank_time(B, cfg, batch, rank, y, steps=20):
    os.environ["LORA_FAKE_WORLD"] = f"{G},{rank},1,0,{y}"
    try:
        c = B.make_config([s.h_in for s in cfg.slots], [s.h_out for s in cfg.slots], [s.n_experts for s in cfg.slots],
                          cfg.rank, cfg.n_adapters, cfg.scale(), batch.n_rows, 0, expert_parallel=True, pp_stages=y,
                          slot_layer=[0] * len(cfg.slots))
        s = B.lora_server_create(c)
    finally:
        del os.environ["LORA_FAKE_WORLD"]
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    B.lora_server_fill_synthetic(s, cfg.seed, st)
    T = batch.n_rows
    xs = {}
    for i, sl in enumerate(cfg.slots):
        if sl.xbuf not in xs:
            x = torch.empty((T, sl.h_in), dtype=torch.int16, device=dev)
            B.lora_synth_fill_rows(x, T, sl.h_in, cfg.seed, li.tag_of(li.KIND_X, sl.xbuf), li.shift_x(), 0, st)
            xs[sl.xbuf] = x
    ys = [torch.zeros((T, sl.h_out), dtype=torch.int16, device=dev) for sl in cfg.slots]
    ad = torch.from_numpy(batch.adapter_ids).to(dev)
    ex = torch.from_numpy(batch.expert_ids).to(dev)
    p = B.lora_plan_create(s, T)
    slots = list(range(len(cfg.slots)))
    xl = [xs[sl.xbuf] for sl in cfg.slots]

    def step(stream):
        B.lora_plan_build(s, p, ad, ex, T, cfg.n_experts, stream)
        B.lora_apply_plan_multi(s, p, slots, xl, ys, B.LORA_BF16, stream)

    g_stream = torch.cuda.Stream()
    g_stream.wait_stream(st)
    with torch.cuda.stream(g_stream):
        step(g_stream)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=g_stream):
            step(g_stream)
    st.wait_stream(g_stream)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(st)
    for k in range(steps):
        graph.replay()
        ev[k + 1].record(st)
    torch.cuda.synchronize()
    times = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    nv = B.lora_plan_stats(s, p)[0]
    B.lora_server_check(s)  # clears the flag raised by the rows other ranks own
    B.lora_plan_destroy(p)
    B.lora_server_destroy(s)
    return float(np.median(times)) * 1e3, int(nv)


def main():
    from paper_2604_07173_b200 import binding as B
    base = li.CONFIGS["mixtral_decode"]
    out = {"what": __doc__.strip().splitlines()[0], "world": G, "adapters": base.n_adapters, "rows": {}}
    link_gbs = 700.0
    row_x = 2 * (4096 + 14336)              # gate/up share x; down has its own
    row_d = 2 * (14336 + 14336 + 4096)      # bf16 deltas of gate, up, down
    for n_tok in (128, 256):
        cfg = li.with_tokens(base, n_tok)
        b = li.make_batch(cfg)
        res = {}
        for x in (1, 2, 4, 8):
            y = G // x
            per_rank = []
            for r in range(x):   # the group of layer 0: ranks 0 .. x-1
                us, rows = rank_time(B, cfg, b, r, y)
                per_rank.append({"rank": r, "us": round(us, 1), "rows": rows})
            own = orc.owner_of(b.adapter_ids, G, 0, None, b.expert_ids, True, y, 0)
            rows_max = int(np.bincount(own[own >= 0], minlength=G).max())
            comm_us = rows_max * (row_x + row_d) / (link_gbs * 1e9) * 1e6
            lora_us = max(p_["us"] for p_ in per_rank)
            res[f"EP{x}-PP{y}"] = {
                "lora_us_measured_slowest_rank": lora_us, "per_rank": per_rank,
                "exchange_us_model": round(comm_us, 1), "sync_scope": x,
                "step_us_model": round(max(lora_us, comm_us), 1)}
        out["rows"][str(n_tok)] = res
        best = min(res, key=lambda k: res[k]["step_us_model"])
        out["rows"][str(n_tok)]["best"] = best
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
