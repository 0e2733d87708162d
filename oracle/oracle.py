"""CPU oracle for the multi-LoRA delta hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product package ``paper_2604_07173_b200`` never imports it and shares no code
with it.  Citations: ``P:n`` = PAPER.md line n (section in brackets).

Functions
- ``segment``            a1: stable sort of valid rows by key a*E+e (R9)
- ``lora_apply_rows``    a2-a4 for a set of rows (plain C loops, fp64, lora_oracle.c)
- ``apply_slot``         convenience: regenerate the touched units of one slot from
                          the seeded generator and run ``lora_apply_rows``
- ``apply_slot_all_rows`` the same over every row of a batch, regenerating at
                          most ``unit_chunk`` units at a time (full-size configs)
- ``shard_dispatch``     the sharded server's dispatch-order rule, so
                          per-rank segment indices can be predicted without GPUs

Pins (tests/test_oracle_pins.py): float64 dense brute force W + s*A*B and its
PEFT transpose, exact-integer probes against numpy int64 matmul, rank-1 outer
products, a hand-worked golden example (tests/golden/), a = -1 zero delta,
permutation equivariance, linearity in s, and for ``segment`` a pure-Python
sorted()+groupby brute force plus hand-written golden cases; ``owner_of`` /
``shard_dispatch`` against a per-row brute force of the routing rule and its
partition / count-matrix invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

import lora_inputs as li

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lora_oracle.c")
_LIB = os.path.join(_HERE, "liblora_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (plain -O2, no -ffast-math, OpenMP over rows)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
               "-ffp-contract=off", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_lora_apply.restype = ctypes.c_int
        lib.oracle_lora_apply.argtypes = [
            ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
            ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
        lib.oracle_round_bf16.restype = ctypes.c_uint16
        lib.oracle_round_bf16.argtypes = [ctypes.c_double]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def round_bf16(d: float) -> int:
    return int(_load().oracle_round_bf16(float(d)))


# ----------------------------------------------------------------------------
# a1: segmentation (reading R9: key a*E+e ascending, ties by row index,
# rows with a = -1 dropped, only non-empty segments)
# ----------------------------------------------------------------------------
def segment(adapter_ids: np.ndarray, expert_ids: Optional[np.ndarray], n_experts: int
            ) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    a = np.asarray(adapter_ids, dtype=np.int64)
    e = np.zeros_like(a) if expert_ids is None else np.asarray(expert_ids, dtype=np.int64)
    valid = np.flatnonzero(a >= 0)
    keys = a[valid] * n_experts + e[valid]
    order = np.argsort(keys, kind="stable")          # textbook stable sort
    perm = valid[order].astype(np.int32)
    sk = keys[order]
    if sk.size == 0:
        return perm, np.zeros(1, np.int32), np.zeros(0, np.int32)
    starts = np.concatenate([[0], np.flatnonzero(sk[1:] != sk[:-1]) + 1])
    seg_offsets = np.concatenate([starts, [sk.size]]).astype(np.int32)
    seg_keys = sk[starts].astype(np.int32)
    return perm, seg_offsets, seg_keys


# ----------------------------------------------------------------------------
# a2-a4: the delta
# ----------------------------------------------------------------------------
def lora_apply_rows(x_bits: np.ndarray, unit_of_row: np.ndarray, scale_of_row: np.ndarray,
                    A_bits: np.ndarray, B_bits: np.ndarray, y: np.ndarray,
                    n_threads: int = 0) -> np.ndarray:
    """y (bf16 bits uint16 or float32) updated in place and returned.

    x_bits [T][h_in] uint16; A_bits [U][h_in][r]; B_bits [U][r][h_out]."""
    lib = _load()
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    T, h_in = x_bits.shape
    A_bits = np.ascontiguousarray(A_bits, dtype=np.uint16)
    B_bits = np.ascontiguousarray(B_bits, dtype=np.uint16)
    U, h_in2, r = A_bits.shape           # shapes hold even when U == 0
    assert h_in2 == h_in and B_bits.shape[0] == U and B_bits.shape[1] == r
    h_out = B_bits.shape[2]
    unit_of_row = np.ascontiguousarray(unit_of_row, dtype=np.int32)
    scale_of_row = np.ascontiguousarray(scale_of_row, dtype=np.float64)
    assert y.shape == (T, h_out) and y.flags.c_contiguous
    if y.dtype == np.float32:
        is32 = 1
    elif y.dtype == np.uint16:
        is32 = 0
    else:
        raise TypeError("y must be float32 or bf16 bits (uint16)")
    rc = lib.oracle_lora_apply(T, h_in, h_out, r, x_bits.ctypes.data, unit_of_row.ctypes.data,
                               scale_of_row.ctypes.data,
                               A_bits.ctypes.data, B_bits.ctypes.data, U,
                               y.ctypes.data, is32, int(n_threads))
    if rc != 0:
        raise ValueError("oracle_lora_apply rejected its arguments")
    return y


def unit_tables(adapter_ids: np.ndarray, expert_ids: Optional[np.ndarray], n_experts: int,
                n_adapters: int, scale: np.ndarray) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Map each row to a compact unit index over the *touched* units.

    Returns (unit_of_row, global_unit_ids, scale_of_row).  Out-of-range ids are
    rejected up front (R10)."""
    a = np.asarray(adapter_ids, dtype=np.int64)
    e = np.zeros_like(a) if expert_ids is None else np.asarray(expert_ids, dtype=np.int64)
    if np.any(a < -1) or np.any(a >= n_adapters):
        raise ValueError("adapter id out of range")
    if np.any((a >= 0) & ((e < 0) | (e >= n_experts))):
        raise ValueError("expert id out of range")
    g = np.where(a >= 0, a * n_experts + e, -1)
    units = np.unique(g[g >= 0])
    unit_of_row = np.where(g >= 0, np.searchsorted(units, g), -1).astype(np.int32)
    scale_of_row = np.where(a >= 0, np.asarray(scale, np.float64)[np.maximum(a, 0)], 0.0)
    return unit_of_row, units.astype(np.int64), scale_of_row


def apply_slot(cfg: li.Config, slot_index: int, batch: li.Batch, rows: Optional[Sequence[int]] = None,
               y0: str = "random", n_threads: int = 0, seed: Optional[int] = None) -> np.ndarray:
    """Oracle y for ``rows`` (default all) of slot ``slot_index`` of ``cfg``.

    Inputs come from lora_inputs' counter-based generator: x rows (xbuf of the
    slot), units (touched only), y0 ("random" or "zero").  Returns y rows as
    float32 (y_dtype fp32) or bf16 bits (bf16)."""
    args = prepare_slot(cfg, slot_index, batch, rows, y0, seed)
    return lora_apply_rows(*args, n_threads=n_threads)


def apply_slot_all_rows(cfg: li.Config, slot_index: int, batch: li.Batch, y0: str = "random",
                        n_threads: int = 0, seed: Optional[int] = None, unit_chunk: int = 256) -> np.ndarray:
    """``apply_slot`` over every row of ``batch`` with bounded host memory.

    The rows are partitioned by their unit (a, e); each call of ``apply_slot``
    covers the rows of at most ``unit_chunk`` distinct units (rows with a = -1
    go with the first call), so at most ``unit_chunk`` units' A/B are
    regenerated at a time (config 5 touches ~2100 units of 5 MB per slot).
    Each row's arithmetic is exactly that of ``lora_apply_rows`` -- only the
    set of rows per call changes -- so the result equals ``apply_slot(cfg,
    slot_index, batch)`` bit for bit (pinned in tests/test_oracle_pins.py)."""
    E = cfg.slots[slot_index].n_experts
    a = batch.adapter_ids.astype(np.int64)
    key = np.where(a >= 0, a * E + batch.expert_ids.astype(np.int64), -1)
    units = np.unique(key[key >= 0])
    chunks = [units[i:i + unit_chunk] for i in range(0, max(units.size, 1), unit_chunk)]
    out = None
    for ci, ch in enumerate(chunks):
        m = np.isin(key, ch)
        if ci == 0:
            m |= key < 0
        rows = np.flatnonzero(m)
        if rows.size == 0:
            continue
        y = apply_slot(cfg, slot_index, batch, rows=rows, y0=y0, n_threads=n_threads, seed=seed)
        if out is None:
            out = np.empty((batch.n_rows, y.shape[1]), y.dtype)
        out[rows] = y
    if out is None:  # empty batch
        out = np.zeros((0, cfg.slots[slot_index].h_out), np.float32 if cfg.y_dtype == "fp32" else np.uint16)
    return out


def prepare_slot(cfg: li.Config, slot_index: int, batch: li.Batch, rows: Optional[Sequence[int]] = None,
                 y0: str = "random", seed: Optional[int] = None):
    """Regenerate the inputs of ``apply_slot`` -> args of ``lora_apply_rows``
    (x, unit_of_row, scale_of_row, A, B, y); lets callers time the oracle's
    arithmetic without the input generation."""
    seed = cfg.seed if seed is None else seed
    slot = cfg.slots[slot_index]
    rows = np.arange(batch.n_rows) if rows is None else np.asarray(rows, dtype=np.int64)
    a = batch.adapter_ids[rows]
    e = batch.expert_ids[rows]
    uor, units, sor = unit_tables(a, e, slot.n_experts, cfg.n_adapters, cfg.scale())
    r = cfg.rank
    A = li.units_A_bits(seed, slot_index, units, slot.h_in, r)
    B = li.units_B_bits(seed, slot_index, units, r, slot.h_out)
    x = li.gen_rows_fast(seed, li.tag_of(li.KIND_X, slot.xbuf), rows, slot.h_in, li.shift_x())
    if y0 == "random":
        y = li.y0_rows_bits(seed, slot_index, rows, slot.h_out)
        if cfg.y_dtype == "fp32":
            y = li.bf16_bits_to_f32(y).copy()
    else:
        y = np.zeros((rows.size, slot.h_out), np.float32 if cfg.y_dtype == "fp32" else np.uint16)
    y = np.ascontiguousarray(y)
    return x, uor, sor, A, B, y


# ----------------------------------------------------------------------------
# sharded server emulation (R18)
# ----------------------------------------------------------------------------
def token_range(n_tokens: int, world: int, rank: int) -> Tuple[int, int]:
    """Rank g holds tokens [g*T/G, (g+1)*T/G) (balanced floor split)."""
    return (n_tokens * rank) // world, (n_tokens * (rank + 1)) // world


def owner_of(adapter_ids: np.ndarray, world: int, n_hot: int = 0, src=None, expert_ids=None,
             ep: bool = False, pp: int = 1, layer: int = 0) -> np.ndarray:
    """Rank that processes each row (R19).

    LoRA Data Parallel stripes the adapters over the G server
    GPUs; adapters [0, n_hot) -- the most popular ones, P:291 -- are
    replicated on every rank, so their rows are processed by the rank that
    holds them (``src``).  Otherwise owner(a) = (a - n_hot) mod G.  Expert
    parallel (``ep``): owner = e mod G.  Hybrid EP_x-PP_y
    (``ep`` with ``pp`` = y > 1): y groups of x = G / y ranks,
    layers interleaved over the groups (layer l -> group l mod y), owner =
    (l mod y) * x + e mod x.  Rows with a = -1 stay at their origin (owner -1)."""
    a = np.asarray(adapter_ids, dtype=np.int64)
    if ep:
        e = np.zeros_like(a) if expert_ids is None else np.asarray(expert_ids, dtype=np.int64)
        x = world // max(pp, 1)
        return np.where(a >= 0, (layer % max(pp, 1)) * x + e % x, -1)
    own = np.where(a >= 0, (a - n_hot) % world, -1)
    if n_hot > 0:
        if src is None:
            raise ValueError("owner_of: replicated adapters need the source rank of each row")
        own = np.where((a >= 0) & (a < n_hot), np.asarray(src, dtype=np.int64), own)
    return own


def shard_dispatch(batch: li.Batch, world: int, n_hot: int = 0, ep: bool = False, pp: int = 1,
                   layer: int = 0) -> List[Dict[str, np.ndarray]]:
    """Per owner rank: the global row indices it receives, in receive order.

    Rows whose owner is their own source rank are processed in place and are
    not exchanged ("local").  Receive order on an owner: by source rank
    ascending, then each source's rows in their original local order.  Also
    returns the send counts matrix ``counts[src][dst]`` (zero diagonal)."""
    k = batch.top_k
    out = []
    src_of_row = np.empty(batch.n_rows, np.int64)
    for g in range(world):
        t0, t1 = token_range(batch.n_tokens, world, g)
        src_of_row[t0 * k:t1 * k] = g
    own = owner_of(batch.adapter_ids, world, n_hot, src_of_row, batch.expert_ids, ep, pp, layer)
    counts = np.zeros((world, world), np.int64)
    for s in range(world):
        for d in range(world):
            if s != d:
                counts[s, d] = int(np.sum((src_of_row == s) & (own == d)))
    for d in range(world):
        recv = []
        for s in range(world):
            if s != d:
                recv.append(np.flatnonzero((src_of_row == s) & (own == d)))
        out.append({"rows": np.concatenate(recv).astype(np.int64) if recv else np.zeros(0, np.int64),
                    "local": np.flatnonzero((src_of_row == d) & (own == d)).astype(np.int64),
                    "counts": counts})
    return out
