"""Shared helpers for the GPU parity tests (not a test module)."""
from __future__ import annotations

import numpy as np
import torch

import lora_inputs as li

DEV = torch.device("cuda", 0)


def binding():
    from paper_2604_07173_b200 import build
    build.build()
    from paper_2604_07173_b200 import binding as B
    return B


def make_server(B, cfg: li.Config, n_slots=None, max_rows=None, fill=True, small_max=None):
    slots = cfg.slots if n_slots is None else cfg.slots[:n_slots]
    c = B.make_config([s.h_in for s in slots], [s.h_out for s in slots], [s.n_experts for s in slots], cfg.rank,
                      cfg.n_adapters, cfg.scale(), max_rows or cfg.n_rows, 0)
    s = B.lora_server_create(c)
    if fill:
        B.lora_server_fill_synthetic(s, cfg.seed)
    if small_max is not None:
        B.lora_server_set_small_seg_max(s, small_max)
    return s


def x_dev(B, cfg: li.Config, slot_index: int, T: int) -> torch.Tensor:
    sl = cfg.slots[slot_index]
    x = torch.empty((T, sl.h_in), dtype=torch.int16, device=DEV)
    B.lora_synth_fill_rows(x, T, sl.h_in, cfg.seed, li.tag_of(li.KIND_X, sl.xbuf), li.shift_x())
    return x


def y0_dev(B, cfg: li.Config, slot_index: int, T: int, kind: str = "random", fp32=None) -> torch.Tensor:
    sl = cfg.slots[slot_index]
    fp32 = (cfg.y_dtype == "fp32") if fp32 is None else fp32
    if kind == "zero":
        return torch.zeros((T, sl.h_out), dtype=torch.float32 if fp32 else torch.int16, device=DEV)
    y = torch.empty((T, sl.h_out), dtype=torch.int16, device=DEV)
    B.lora_synth_fill_rows(y, T, sl.h_out, cfg.seed, li.tag_of(li.KIND_Y0, slot_index), li.shift_y0())
    if fp32:
        y = (y.to(torch.int32) << 16).view(torch.float32)
        y = y.contiguous()
    return y


def register(B, sh, bufs):
    """Register device buffers (x / y) of a sharded server for the push path."""
    B.lora_shard_register(sh, bufs, [t.numel() * t.element_size() for t in bufs])


def ids_dev(batch: li.Batch):
    return (torch.from_numpy(batch.adapter_ids).to(DEV), torch.from_numpy(batch.expert_ids).to(DEV))


def as_float(y) -> np.ndarray:
    """GPU y (fp32 or bf16-bits int16) or oracle y (f32 / uint16 bits) -> float64 numpy."""
    if isinstance(y, torch.Tensor):
        y = y.detach().cpu()
        if y.dtype == torch.float32:
            return y.numpy().astype(np.float64)
        return li.bf16_bits_to_f32(y.numpy().view(np.uint16)).astype(np.float64)
    if y.dtype == np.uint16:
        return li.bf16_bits_to_f32(y).astype(np.float64)
    return y.astype(np.float64)


def assert_parity(got, ref, what=""):
    """North-star bound: max|err| <= 1e-2 * max|y_ref| + 1e-3 (R12)."""
    g, r = as_float(got), as_float(ref)
    assert g.shape == r.shape, (g.shape, r.shape)
    err = float(np.abs(g - r).max()) if g.size else 0.0
    tol = 1e-2 * float(np.abs(r).max() if r.size else 0.0) + 1e-3
    assert err <= tol, f"{what}: max|err| {err:.4e} > tol {tol:.4e}"
    return err, tol


def sample_rows(batch: li.Batch, n: int, seed: int = 0, E: int = 1) -> np.ndarray:
    """Rows covering the largest segment, singletons, no-LoRA rows and a random tail."""
    rng = np.random.default_rng(seed)
    a = batch.adapter_ids.astype(np.int64)
    key = np.where(a >= 0, a * E + batch.expert_ids, -1)
    valid = np.flatnonzero(key >= 0)
    uniq, cnt = np.unique(key[valid], return_counts=True)
    picks = set()
    big = uniq[np.argmax(cnt)]
    picks.update(np.flatnonzero(key == big)[:8].tolist())
    single = uniq[cnt == 1][:8]
    for k in single:
        picks.update(np.flatnonzero(key == k).tolist())
    picks.update(np.flatnonzero(key < 0)[:2].tolist())
    picks.add(batch.n_rows - 1)
    rest = rng.choice(batch.n_rows, size=min(batch.n_rows, n), replace=False)
    for r in rest:
        if len(picks) >= n:
            break
        picks.add(int(r))
    return np.array(sorted(picks), dtype=np.int64)
