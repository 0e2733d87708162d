"""Randomised parity sweep (GPU): random slot shapes, ranks, expert counts,
adapter counts, batch sizes, id distributions, y dtypes and kernel routes
(CUDA cores only / tcgen05 forced / mixed) and entry points (in-place apply,
delta API, the sharded push path's G = 1 loopback), each compared element by
element with the CPU oracle.  Not part of the default suite (minutes of oracle time);

    python tools/fuzz_parity.py [n_cases] [seed]

Prints one line per case and a summary; exits 1 on the first mismatch.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import lora_inputs as li  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from tests import gpu_util as U  # noqa: E402


def one_case(B, rng, k):
    rank = int(rng.choice([8, 16, 32, 64, 128]))
    E = int(rng.choice([1, 2, 4, 8]))
    top_k = 1 if E == 1 else int(rng.choice([1, 2]))
    n_slots = int(rng.integers(1, 4))
    widths = [128, 256, 384, 512, 768, 1024, 2048]
    slots = []
    for i in range(n_slots):
        h_in = int(rng.choice(widths))
        h_out = int(rng.choice(widths))
        xbuf = i if rng.random() < 0.7 or i == 0 else slots[-1].xbuf
        if xbuf != i:
            h_in = slots[-1].h_in
        slots.append(li.Slot(f"s{i}", h_in, h_out, E, xbuf))
    n_ad = int(rng.choice([3, 16, 64, 300]))
    n_tok = int(rng.choice([1, 7, 64, 300, 1500, 2600, 9000]))
    y_dtype = "fp32" if rng.random() < 0.4 else "bf16"
    n_seqs = int(rng.choice([0, 0, 2, 8])) if n_tok >= 8 else 0
    zipf = float(rng.choice([0.0, 1.2, 2.0]))
    cfg = li.Config(f"fuzz{k}", 100 + k, tuple(slots), rank, n_ad, E, top_k, n_tok, y_dtype, zipf_s=zipf,
                    n_seqs=n_seqs, no_lora_frac=float(rng.choice([0.0, 0.1])))
    route = str(rng.choice(["default", "tc", "simt", "tc_all"]))
    api = str(rng.choice(["apply", "apply", "delta", "push_loopback"]))
    os.environ["LORA_TC_MIN_ROWS"] = "0" if route in ("tc", "tc_all") else os.environ.get("FUZZ_MIN_ROWS", "256")
    b = li.make_batch(cfg)
    small = {"default": None, "tc": 4, "simt": -1, "tc_all": 0}[route]
    s = U.make_server(B, cfg, small_max=small)
    try:
        T = b.n_rows
        ad, ex = U.ids_dev(b)
        xs = {}
        for i, sl in enumerate(cfg.slots):
            if sl.xbuf not in xs:
                xs[sl.xbuf] = U.x_dev(B, cfg, i, T)
        dt = B.LORA_FP32 if y_dtype == "fp32" else B.LORA_BF16
        y0 = "zero" if api == "delta" else "random"
        ys = [U.y0_dev(B, cfg, i, T, y0) for i in range(n_slots)]
        p = B.lora_plan_create(s, T)
        B.lora_plan_build(s, p, ad, ex if E > 1 else None, T, E)
        stats = B.lora_plan_stats(s, p)
        xl = [xs[sl.xbuf] for sl in cfg.slots]
        if api == "delta":
            B.lora_apply_plan_multi_delta(s, p, list(range(n_slots)), xl, ys, dt)
        elif api == "push_loopback":
            os.environ["LORA_SHARD_LOOPBACK"] = "1"
            c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                              [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(), T, 0)
            sh = B.lora_server_create_sharded(c, 0, 1, B.lora_nccl_unique_id())
            try:
                B.lora_server_fill_synthetic(sh, cfg.seed)
                xd = [x.clone() for x in xl]  # one registered buffer per slot
                U.register(B, sh, xd + ys)
                B.lora_apply_sharded(sh, list(range(n_slots)), xd, ad, ex if E > 1 else None, ys, dt, T)
                torch.cuda.synchronize()
                assert B.lora_server_check(sh) == B.LORA_OK
            finally:
                B.lora_server_destroy(sh)
                del os.environ["LORA_SHARD_LOOPBACK"]
        else:
            B.lora_apply_plan_multi(s, p, list(range(n_slots)), xl, ys, dt)
        torch.cuda.synchronize()
        assert B.lora_server_check(s) == B.LORA_OK
        B.lora_plan_destroy(p)
        for i in range(n_slots):
            U.assert_parity(ys[i], orc.apply_slot(cfg, i, b, y0=y0), f"case {k} slot {i}")
        print(f"case {k}: r={rank} E={E} top{top_k} slots={[(sl.h_in, sl.h_out) for sl in cfg.slots]} "
              f"adapters={n_ad} tokens={n_tok} seqs={n_seqs} zipf={zipf} y={y_dtype} route={route} api={api} "
              f"plan(valid,segs,groups,tiles)={tuple(stats)} OK", flush=True)
    finally:
        B.lora_server_destroy(s)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    B = U.binding()
    rng = np.random.default_rng(seed)
    for k in range(n):
        one_case(B, rng, k)
    print(f"fuzz: {n} cases OK")


if __name__ == "__main__":
    main()
