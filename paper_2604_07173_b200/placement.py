"""Popularity-aware adapter placement for the Sharded LoRA Server (host logic).

LoRA Data Parallel stripes the adapters over the G server GPUs (P:288-291,
Sec. 4.1); under skewed popularity the owner of a hot adapter receives a large
share of all activations.  The library therefore accepts
``n_replicated = h``: adapters [0, h) -- ids ordered by popularity -- are
stored on every rank and their rows are processed where they are, the rest is
owned by rank (a - h) mod G (include/lora_server.h, R19).

Replication trades HBM traffic (each rank reads the hot units its rows touch)
for less exchange and a balanced load.  ``choose_n_replicated`` picks h from
the observed ids with a per-rank bytes model -- the same rule the library
applies, written out on the host -- and returns the cost table it used.
"""
from __future__ import annotations

from typing import Dict, Iterable, Optional, Sequence

import numpy as np


def owner(adapter_ids: np.ndarray, world: int, n_hot: int, src: np.ndarray, expert_ids=None,
          ep: bool = False) -> np.ndarray:
    """Rank that processes each row (-1 for rows without an adapter).  ep:
    expert parallel, owner = e mod world (include/lora_server.h)."""
    a = np.asarray(adapter_ids, np.int64)
    if ep:
        e = np.zeros_like(a) if expert_ids is None else np.asarray(expert_ids, np.int64)
        return np.where(a >= 0, e % world, -1)
    own = np.where(a >= 0, (a - n_hot) % world, -1)
    return np.where((a >= 0) & (a < n_hot), np.asarray(src, np.int64), own)


def rank_hbm_bytes(adapter_ids: np.ndarray, expert_ids: Optional[np.ndarray], src: np.ndarray, world: int,
                   n_hot: int, unit_bytes: float, row_bytes: float, ep: bool = False) -> np.ndarray:
    """Algorithmic HBM bytes per rank of one sharded apply (SURVEY 8d per
    rank): each unit the rank serves read once, each row it serves read and
    written once, each of its rows served elsewhere accumulated once."""
    a = np.asarray(adapter_ids, np.int64)
    e = np.zeros_like(a) if expert_ids is None else np.asarray(expert_ids, np.int64)
    src = np.asarray(src, np.int64)
    own = owner(a, world, n_hot, src, e, ep)
    valid = a >= 0
    n_e = int(e.max()) + 1 if e.size else 1
    key = a * n_e + e
    out = np.zeros(world)
    for g in range(world):
        mine = valid & (own == g)
        remote_out = int(np.sum(valid & (src == g) & (own != g)))
        out[g] = np.unique(key[mine]).size * unit_bytes + int(mine.sum()) * row_bytes + remote_out * row_bytes
    return out


def rank_costs(adapter_ids: np.ndarray, expert_ids: Optional[np.ndarray], src: np.ndarray, world: int, n_hot: int,
               unit_bytes: float, row_bytes: float, xfer_bytes: float, hbm_gbs: float = 6500.0,
               link_gbs: float = 700.0, ep: bool = False) -> np.ndarray:
    """Modelled time (s) per rank of one sharded apply on the NCCL path
    (unregistered buffers: staged send / receive, not overlapped).

    unit_bytes: weight bytes of one (adapter, expert) unit over all slots;
    row_bytes: HBM bytes per processed row (x read, y or delta write);
    xfer_bytes: bytes one remote row moves over NVLink (x out + delta back)."""
    a = np.asarray(adapter_ids, np.int64)
    e = np.zeros_like(a) if expert_ids is None else np.asarray(expert_ids, np.int64)
    src = np.asarray(src, np.int64)
    own = owner(a, world, n_hot, src, e, ep)
    valid = a >= 0
    n_e = int(e.max()) + 1 if e.size else 1
    key = a * n_e + e
    out = np.zeros(world)
    for g in range(world):
        mine = valid & (own == g)
        units = np.unique(key[mine]).size
        remote_in = int(np.sum(mine & (src != g)))
        remote_out = int(np.sum(valid & (src == g) & (own != g)))
        hbm = units * unit_bytes + int(mine.sum()) * row_bytes + remote_out * row_bytes
        # NVLink is full duplex: sends and receives overlap
        out[g] = hbm / (hbm_gbs * 1e9) + max(remote_in, remote_out) * xfer_bytes / (link_gbs * 1e9)
    return out


def rank_costs_push(adapter_ids: np.ndarray, expert_ids: Optional[np.ndarray], src: np.ndarray, world: int,
                    n_hot: int, unit_bytes: float, row_bytes: float, x_bytes: float, d_bytes: float,
                    hbm_gbs: float = 6500.0, link_gbs: float = 700.0, fixed_s: float = 40e-6, ep: bool = False,
                    pp: int = 1, layer: int = 0) -> np.ndarray:
    """Modelled time (s) per rank of one sharded apply on the push path
    (registered buffers; include/lora_server.h lora_apply_sharded).

    The owner's shrink reads each received row's x from the source's HBM and
    its expand red.adds the delta into the source's y, so a row's x read and
    y read-modify-write always hit its SOURCE's HBM: rank g's HBM bytes are
    its served units' weights plus all of its own rows (row_bytes each),
    wherever they are computed.  NVLink carries x in and deltas out of each
    owner (x_bytes + d_bytes per exchanged row, full duplex).  Both transfers
    are fused into the kernels, so they overlap the weight stream: time =
    max(HBM time, link time) + fixed_s (bucket / announce / recv-prep /
    owner-side segmentation / done + wait: the measured protocol overhead)."""
    a = np.asarray(adapter_ids, np.int64)
    e = np.zeros_like(a) if expert_ids is None else np.asarray(expert_ids, np.int64)
    src = np.asarray(src, np.int64)
    if ep and pp > 1:
        x = world // pp
        own = np.where(a >= 0, (layer % pp) * x + e % x, -1)
    else:
        own = owner(a, world, n_hot, src, e, ep)
    valid = a >= 0
    n_e = int(e.max()) + 1 if e.size else 1
    key = a * n_e + e
    out = np.zeros(world)
    for g in range(world):
        mine = valid & (own == g)
        units = np.unique(key[mine]).size
        hbm = units * unit_bytes + int(np.sum(valid & (src == g))) * row_bytes
        rin = int(np.sum(mine & (src != g)))
        rout = int(np.sum(valid & (src == g) & (own != g)))
        link_in = rin * x_bytes + rout * d_bytes
        link_out = rout * x_bytes + rin * d_bytes
        out[g] = max(hbm / (hbm_gbs * 1e9), max(link_in, link_out) / (link_gbs * 1e9)) + fixed_s
    return out


def _cost(adapter_ids, expert_ids, src, world, h, unit_bytes, row_bytes, xfer_bytes, x_bytes, d_bytes, ep=False,
          **kw) -> float:
    """Slowest rank's modelled time: the push path's model when the x / delta
    split is given (x_bytes, d_bytes), else the NCCL path's."""
    if x_bytes is not None:
        return float(rank_costs_push(adapter_ids, expert_ids, src, world, h, unit_bytes, row_bytes, x_bytes, d_bytes,
                                     ep=ep, **kw).max())
    return float(rank_costs(adapter_ids, expert_ids, src, world, h, unit_bytes, row_bytes, xfer_bytes, ep=ep,
                            **kw).max())


def choose_n_replicated(adapter_ids: np.ndarray, expert_ids: Optional[np.ndarray], src: np.ndarray, world: int,
                        unit_bytes: float, row_bytes: float, xfer_bytes: float,
                        candidates: Optional[Iterable[int]] = None, x_bytes: Optional[float] = None,
                        d_bytes: Optional[float] = None, **kw) -> Dict:
    """Pick h minimising the slowest rank's modelled time; ties -> smaller h."""
    if world <= 1:
        return {"n_replicated": 0, "table": {0: 0.0}}
    n_ad = int(np.max(adapter_ids)) + 1 if np.size(adapter_ids) else 0
    if candidates is None:
        candidates = [0] + [1 << i for i in range(12) if (1 << i) <= max(n_ad, 1)]
    table = {}
    for h in candidates:
        table[int(h)] = _cost(adapter_ids, expert_ids, src, world, int(h), unit_bytes, row_bytes, xfer_bytes,
                              x_bytes, d_bytes, **kw)
    best = min(table, key=lambda h: (table[h], h))
    return {"n_replicated": best, "table": table}


def choose_placement(adapter_ids: np.ndarray, expert_ids: Optional[np.ndarray], src: np.ndarray, world: int,
                     unit_bytes: float, row_bytes: float, xfer_bytes: float, x_bytes: Optional[float] = None,
                     d_bytes: Optional[float] = None, **kw) -> Dict:
    """Best of LoRA Data Parallel with replication (choose_n_replicated) and
    expert parallel (MoE only), by the slowest rank's modelled time."""
    dp = choose_n_replicated(adapter_ids, expert_ids, src, world, unit_bytes, row_bytes, xfer_bytes,
                             x_bytes=x_bytes, d_bytes=d_bytes, **kw)
    out = {"expert_parallel": False, "n_replicated": dp["n_replicated"], "table": dict(dp["table"])}
    if world > 1 and expert_ids is not None:
        t_ep = _cost(adapter_ids, expert_ids, src, world, 0, unit_bytes, row_bytes, xfer_bytes, x_bytes, d_bytes,
                     ep=True, **kw)
        out["table"]["ep"] = t_ep
        if t_ep < dp["table"][dp["n_replicated"]]:
            out.update(expert_parallel=True, n_replicated=0)
    return out


def hybrid_table(adapter_ids: np.ndarray, expert_ids: np.ndarray, src: np.ndarray, world: int, unit_bytes: float,
                 row_bytes: float, x_bytes: float, d_bytes: float, layer: int = 0, **kw) -> Dict[str, float]:
    """Slowest rank's modelled time (push path) of one layer's apply under
    every EP_x-PP_y layout with x * y = world (Table-BD
    compares EP1-PP8 / EP2-PP4 / EP4-PP2 / EP8-PP1 at 8 GPUs).  Under PP the
    ranks of the other groups serve nothing for this layer (they run other
    layers for other instances), so the layer's time is its group's."""
    out = {}
    for y in [d for d in range(1, world + 1) if world % d == 0][::-1]:
        x = world // y
        out[f"EP{x}-PP{y}"] = float(rank_costs_push(adapter_ids, expert_ids, src, world, 0, unit_bytes, row_bytes,
                                                    x_bytes, d_bytes, ep=True, pp=y, layer=layer, **kw).max())
    return out


def slot_bytes_push(h_in: Sequence[int], h_out: Sequence[int], xbuf: Sequence[int], rank: int, y_bytes: int,
                    delta_bytes: int):
    """(unit_bytes, row_bytes, x_bytes, d_bytes) for the push model: x_bytes
    the distinct x rows one exchanged row reads over NVLink, d_bytes its
    deltas pushed back (bf16 for a bf16 y)."""
    unit, row, _ = slot_bytes(h_in, h_out, xbuf, rank, y_bytes, delta_bytes)
    seen, x_b = set(), 0
    for hi, xb in zip(h_in, xbuf):
        if xb not in seen:
            seen.add(xb)
            x_b += 2 * hi
    return unit, row, float(x_b), float(sum(delta_bytes * ho for ho in h_out))


def sources_of_rows(n_tokens: int, top_k: int, world: int) -> np.ndarray:
    """Source rank of each token-major row when rank g holds tokens
    [g*T/G, (g+1)*T/G) (the bench's and the tests' split)."""
    src = np.empty(n_tokens * top_k, np.int64)
    for g in range(world):
        t0, t1 = (n_tokens * g) // world, (n_tokens * (g + 1)) // world
        src[t0 * top_k:t1 * top_k] = g
    return src


def slot_bytes(h_in: Sequence[int], h_out: Sequence[int], xbuf: Sequence[int], rank: int, y_bytes: int,
               delta_bytes: int):
    """(unit_bytes, row_bytes, xfer_bytes) for a slot list (bf16 weights and x)."""
    unit = sum(2 * rank * (hi + ho) for hi, ho in zip(h_in, h_out))
    seen, x_b = set(), 0
    for hi, xb in zip(h_in, xbuf):
        if xb not in seen:
            seen.add(xb)
            x_b += 2 * hi
    row = x_b + sum(2 * y_bytes * ho for ho in h_out)
    xfer = x_b + sum(delta_bytes * ho for ho in h_out)
    return float(unit), float(row), float(xfer)
