#!/usr/bin/env python
"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Cases (each checked against the oracle, so a sanitizer-clean run is also a
correct one):
  tiny      one MoE slot, r = 8, fp32 y (CUDA-core chain)
  mid       two slots, r = 64, bf16 y, segments on both chains, concurrent
            (tcgen05 chain on the side stream)
  mid_fp32  the same with an fp32 y (direct tcgen05 epilogue)
  wholek    4100 rows: multi-CTA segmenter, whole-K tcgen05 shrink
  llama     r = 16, 8 slots (resolver warps, staged-tile expand)
  tc16 / tc32 / tc128   the mid config at r = 16 / 32 / 128 with the tcgen05
            chain forced on (SWIZZLE_32B / 64B operands; r = 128: two K blocks,
            Bt re-tiled by cp.async in the expand's producer warp)
  push      sharded server at G = 1, loopback through the push path
            (announce / recv-prep / device-T segmenter / remote-x shrink /
            red.add expand / done + wait)
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


def _mid(rank=64, n_tok=300, y="bf16"):
    return li.Config("mid", 8, (li.Slot("a", 512, 768, 4, 0), li.Slot("b", 768, 512, 4, 1)), rank, 24, 4, 2,
                     n_tok, y)


def run_unsharded(B, cfg, slots, name):
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        T = b.n_rows
        ad, ex = U.ids_dev(b)
        E = cfg.slots[slots[0]].n_experts
        xs = {}
        for i in slots:
            if cfg.slots[i].xbuf not in xs:
                xs[cfg.slots[i].xbuf] = U.x_dev(B, cfg, i, T)
        ys = [U.y0_dev(B, cfg, i, T) for i in slots]
        p = B.lora_plan_create(s, T)
        B.lora_plan_build(s, p, ad, ex if E > 1 else None, T, E)
        B.lora_apply_plan_multi(s, p, slots, [xs[cfg.slots[i].xbuf] for i in slots], ys,
                                B.LORA_FP32 if cfg.y_dtype == "fp32" else B.LORA_BF16)
        torch.cuda.synchronize()
        assert B.lora_server_check(s) == B.LORA_OK
        B.lora_plan_destroy(p)
        for j, i in enumerate(slots):
            U.assert_parity(ys[j], orc.apply_slot(cfg, i, b), f"{name} slot {i}")
    finally:
        B.lora_server_destroy(s)


def run_push(B):
    os.environ["LORA_SHARD_LOOPBACK"] = "1"
    cfg = _mid()
    b = li.make_batch(cfg)
    T = b.n_rows
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots], [4, 4], cfg.rank,
                      cfg.n_adapters, cfg.scale(), T, 0)
    sh = B.lora_server_create_sharded_host(c, 0, 1, lambda d: d)
    try:
        B.lora_server_fill_synthetic(sh, cfg.seed)
        ad, ex = U.ids_dev(b)
        xs = [U.x_dev(B, cfg, i, T) for i in range(2)]
        ys = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        U.register(B, sh, xs + ys)
        B.lora_apply_sharded(sh, [0, 1], xs, ad, ex, ys, B.LORA_BF16, T)
        torch.cuda.synchronize()
        assert B.lora_server_check(sh) == B.LORA_OK
        for i in range(2):
            U.assert_parity(ys[i], orc.apply_slot(cfg, i, b), f"push slot {i}")
    finally:
        B.lora_server_destroy(sh)
        del os.environ["LORA_SHARD_LOOPBACK"]


def main():
    B = U.binding()
    cases = sys.argv[1:] or ["tiny", "mid", "mid_fp32", "wholek", "llama", "tc16", "tc32", "tc128", "push"]
    for c in cases:
        if c == "tiny":
            run_unsharded(B, li.CONFIGS["tiny"], [0], c)
        elif c == "mid":
            run_unsharded(B, _mid(), [0, 1], c)
        elif c == "mid_fp32":
            run_unsharded(B, _mid(y="fp32"), [0, 1], c)
        elif c == "wholek":
            run_unsharded(B, _mid(n_tok=2050), [0, 1], c)
        elif c == "llama":
            cfg = li.CONFIGS["llama_decode"]
            cfg = li.Config("llama8", 2, cfg.slots[:8], 16, 128, 1, 1, 256, "bf16")
            run_unsharded(B, cfg, list(range(8)), c)
        elif c in ("tc16", "tc32", "tc128"):
            os.environ["LORA_TC_MIN_ROWS"] = "0"
            run_unsharded(B, _mid(rank=int(c[2:])), [0, 1], c)
            del os.environ["LORA_TC_MIN_ROWS"]
        elif c == "push":
            run_push(B)
        print(f"sanitize case {c}: OK", flush=True)


if __name__ == "__main__":
    main()
