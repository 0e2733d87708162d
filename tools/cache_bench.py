"""Resident-adapter cache: host->device load throughput and layer-wise overlap.

Mixtral-shaped slots for L layers x {gate, up, down} (r 64, E 8), 64 adapters,
n_resident 8.  Each step requires 8 new adapters (every weight reloaded) and
applies the layers one by one on the same stream:
  overlapped  -- lora_server_require, then per-layer applies (each waits only
                 for its own layer's copies);
  serialized  -- the same, with a stream synchronize after require.
Prints GB/s of the weight copies and the time of both variants.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import lora_inputs as li
from paper_2604_07173_b200 import binding as B

L, NAD, NRES, TOK = 4, 64, 8, 2048
slots = []
for l in range(L):
    slots += [li.Slot(f"L{l}.gate", 4096, 14336, 8, 2 * l), li.Slot(f"L{l}.up", 4096, 14336, 8, 2 * l),
              li.Slot(f"L{l}.down", 14336, 4096, 8, 2 * l + 1)]
cfg = li.Config("cache_bench", 9, tuple(slots), 64, NAD, 8, 2, TOK, "bf16")
T = TOK * 2
c = B.make_config([s.h_in for s in slots], [s.h_out for s in slots], [8] * len(slots), 64, NAD, cfg.scale(), T, 0,
                  n_resident=NRES)
s = B.lora_server_create(c)
B.lora_server_fill_synthetic(s, cfg.seed)
stream = torch.cuda.current_stream()
xs = {}
for i, sl in enumerate(slots):
    if sl.xbuf not in xs:
        xs[sl.xbuf] = B_x = torch.empty((T, sl.h_in), dtype=torch.int16, device="cuda")
        B.lora_synth_fill_rows(B_x, T, sl.h_in, cfg.seed, li.tag_of(li.KIND_X, sl.xbuf), li.shift_x(), 0, stream)
ys = [torch.zeros((T, sl.h_out), dtype=torch.int16, device="cuda") for sl in slots]
rng = np.random.default_rng(0)
per_adapter = sum(8 * 64 * (sl.h_in + sl.h_out) * 2 for sl in slots)
plan = B.lora_plan_create(s, T)


def step(k, serialize):
    sub = np.arange(NRES) + (k % (NAD // NRES)) * NRES   # a fresh set each step
    a = torch.from_numpy(rng.choice(sub, T).astype(np.int32)).cuda()
    e = torch.from_numpy(rng.integers(0, 8, T).astype(np.int32)).cuda()
    n = B.lora_server_require(s, sub, stream)
    if serialize:
        torch.cuda.synchronize()
    B.lora_plan_build(s, plan, a, e, T, 8, stream)
    for l in range(L):
        idx = [3 * l, 3 * l + 1, 3 * l + 2]
        B.lora_apply_plan_multi(s, plan, idx, [xs[slots[i].xbuf] for i in idx], [ys[i] for i in idx], B.LORA_BF16,
                                stream)
    return n


for mode in (False, True, False, True):
    for k in range(2):
        step(k, mode)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loads = 0
    for k in range(2, 10):
        loads += step(k, mode)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 8
    print(f"{'serialized' if mode else 'overlapped'}: {dt * 1e3:.2f} ms/step, {loads / 8:.0f} adapters loaded/step, "
          f"{loads / 8 * per_adapter / 1e9:.2f} GB/step -> {loads / 8 * per_adapter / dt / 1e9:.1f} GB/s", flush=True)
B.lora_plan_destroy(plan)
B.lora_server_destroy(s)
