"""Seeded synthetic inputs for the multi-LoRA delta hot path.

This module is the ONE piece shared by the oracle (``oracle/``) and the CUDA
path (``paper_2604_07173_b200``): it only draws numbers.  It contains none of
the method's arithmetic (no shrink, expand, scale or sort) -- see DESIGN.md
"Input recipe".

Contents
- ``CONFIGS``: the five BASELINE.json configurations.
- ``zipf_probs`` / ``make_batch``: per-row adapter ids (Zipf s=1.2) and
  per-row expert ids (top-k distinct uniform), token-major rows ``t*k + j``
  ("b x k" routed activations).
- ``hash_u64`` / ``hash_bf16_bits``: a counter-based generator for every
  floating-point tensor (weights, activations, base outputs).  The CUDA side
  implements the *same* counter-based generator in its synthetic-fill kernel
  (csrc/synth_fill.cu); the two share no code, only this written recipe:

      mix64(z)  = splitmix64 finaliser
      base      = mix64(seed*G ^ tag*T ^ major*M)             (mod 2^64)
      h         = mix64(base + minor*G)
      q         = (h >> 56) - 128                              (int in [-128,127])
      value     = q * 2^-shift                                 (exact in bf16)

  Every generated value has <= 8 significant bits, so it is exactly
  representable in bf16 and fp32; no rounding is involved anywhere.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# ----------------------------------------------------------------------------
# counter-based generator
# ----------------------------------------------------------------------------
U64 = np.uint64
_G = U64(0x9E3779B97F4A7C15)   # golden-ratio increment (splitmix64)
_T = U64(0xD1B54A32D192ED03)
_M = U64(0xC2B2AE3D27D4EB4F)
_C1 = U64(0xBF58476D1CE4E5B9)
_C2 = U64(0x94D049BB133111EB)

# tensor kinds used in the ``tag`` (tag = kind << 16 | index)
KIND_A, KIND_B, KIND_X, KIND_Y0 = 1, 2, 3, 4


def tag_of(kind: int, index: int) -> int:
    return (int(kind) << 16) | int(index)


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=U64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> U64(30))) * _C1
        z = (z ^ (z >> U64(27))) * _C2
    return z ^ (z >> U64(31))


def hash_base(seed: int, tag: int, major) -> np.ndarray:
    major = np.asarray(major, dtype=U64)
    with np.errstate(over="ignore"):
        z = (U64(seed) * _G) ^ (U64(tag) * _T) ^ (major * _M)
    return mix64(z)


def hash_u64(seed: int, tag: int, major, minor) -> np.ndarray:
    base = hash_base(seed, tag, major)
    minor = np.asarray(minor, dtype=U64)
    with np.errstate(over="ignore"):
        return mix64(base + minor * _G)


def hash_q(seed: int, tag: int, major, minor) -> np.ndarray:
    """int32 in [-128, 127]"""
    h = hash_u64(seed, tag, major, minor)
    return (h >> U64(56)).astype(np.int32) - 128


def hash_bf16_bits(seed: int, tag: int, major, minor, shift: int) -> np.ndarray:
    """bf16 bit patterns (uint16) of q * 2^-shift."""
    q = hash_q(seed, tag, major, minor).astype(np.float32)
    f = (q * np.float32(2.0 ** -shift)).astype(np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16_bits_exact(f: np.ndarray) -> np.ndarray:
    """Truncating cast; callers only pass values already exact in bf16."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    u = f.view(np.uint32)
    if np.any(u & np.uint32(0xFFFF)):
        raise ValueError("value not exactly representable in bf16")
    return (u >> np.uint32(16)).astype(np.uint16)


# value scales (powers of two so the values stay exact)
def shift_x() -> int:
    return 6          # x in [-2, 2), std ~1.15


def shift_y0() -> int:
    return 6


def shift_A(h_in: int) -> int:
    return 7 + int(math.ceil(math.log2(h_in) / 2.0))    # std ~ 0.577/sqrt(h_in)


def shift_B(r: int) -> int:
    return 7 + int(math.ceil(math.log2(r) / 2.0))       # std ~ 0.577/sqrt(r)


def unit_A_bits(seed: int, slot: int, unit: int, h_in: int, r: int) -> np.ndarray:
    """A_{a,e} of one unit in the paper's orientation, bf16 bits [h_in][r].

    minor index = j*r + k for element A[j, k]."""
    minor = np.arange(h_in * r, dtype=U64)
    return hash_bf16_bits(seed, tag_of(KIND_A, slot), unit, minor, shift_A(h_in)).reshape(h_in, r)


def unit_B_bits(seed: int, slot: int, unit: int, r: int, h_out: int) -> np.ndarray:
    """B_{a,e} of one unit, bf16 bits [r][h_out]; minor = k*h_out + c."""
    minor = np.arange(r * h_out, dtype=U64)
    return hash_bf16_bits(seed, tag_of(KIND_B, slot), unit, minor, shift_B(r)).reshape(r, h_out)


_CGEN = None


def _cgen():
    """Compiled copy of the same generator (lora_inputs/_gen.c), for large sets."""
    global _CGEN
    if _CGEN is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, so = os.path.join(here, "_gen.c"), os.path.join(here, "_gen.so")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-o", so, src])
        lib = ctypes.CDLL(so)
        lib.gen_bf16_rows.restype = None
        lib.gen_bf16_rows.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]
        _CGEN = lib
    return _CGEN


def gen_rows_fast(seed: int, tag: int, majors: Sequence[int], n_minor: int, shift: int) -> np.ndarray:
    """bf16 bits [len(majors)][n_minor], minor = 0..n_minor-1 (C generator)."""
    majors = np.ascontiguousarray(np.asarray(majors, dtype=np.uint64))
    out = np.empty((majors.size, n_minor), np.uint16)
    _cgen().gen_bf16_rows(int(seed), int(tag), majors.ctypes.data, majors.size, n_minor, int(shift),
                          out.ctypes.data)
    return out


def units_A_bits(seed: int, slot: int, units: Sequence[int], h_in: int, r: int) -> np.ndarray:
    """Stack of unit_A_bits for many units: [U][h_in][r]."""
    return gen_rows_fast(seed, tag_of(KIND_A, slot), units, h_in * r, shift_A(h_in)).reshape(-1, h_in, r)


def units_B_bits(seed: int, slot: int, units: Sequence[int], r: int, h_out: int) -> np.ndarray:
    return gen_rows_fast(seed, tag_of(KIND_B, slot), units, r * h_out, shift_B(r)).reshape(-1, r, h_out)


def rows_bits(seed: int, kind: int, index: int, rows: Sequence[int], width: int, shift: int) -> np.ndarray:
    """bf16 bits [len(rows)][width] of an activation-like tensor; major = row id."""
    rows = np.asarray(rows, dtype=U64).reshape(-1, 1)
    minor = np.arange(width, dtype=U64).reshape(1, -1)
    return hash_bf16_bits(seed, tag_of(kind, index), rows, minor, shift)


def x_rows_bits(seed: int, xbuf: int, rows: Sequence[int], h_in: int) -> np.ndarray:
    return rows_bits(seed, KIND_X, xbuf, rows, h_in, shift_x())


def y0_rows_bits(seed: int, slot: int, rows: Sequence[int], h_out: int) -> np.ndarray:
    return rows_bits(seed, KIND_Y0, slot, rows, h_out, shift_y0())


# ----------------------------------------------------------------------------
# configurations (BASELINE.json "configs")
# ----------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Slot:
    name: str
    h_in: int
    h_out: int
    n_experts: int
    xbuf: int          # which activation buffer feeds this slot (gate/up share one)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    index: int
    slots: Tuple[Slot, ...]
    rank: int
    n_adapters: int
    n_experts: int
    top_k: int
    n_tokens: int
    y_dtype: str                # "fp32" or "bf16"
    zipf_s: float = 1.2
    n_seqs: int = 0             # prefill: adapters drawn per sequence, not per token
    no_lora_frac: float = 0.0   # fraction of tokens with adapter id -1

    @property
    def n_rows(self) -> int:
        return self.n_tokens * self.top_k

    @property
    def seed(self) -> int:
        return 1000 + self.index

    def scale(self) -> np.ndarray:
        """Per-adapter s_a in {0.5, 1, 2} by a mod 3 (reading R1)."""
        return np.array([(0.5, 1.0, 2.0)[a % 3] for a in range(self.n_adapters)], dtype=np.float32)


def _moe_slots(layer: int = 0) -> Tuple[Slot, ...]:
    # Mixtral-8x7B: hidden 4096, FFN 14336, 8 experts (public config)
    b = 3 * layer
    return (Slot(f"L{layer}.gate", 4096, 14336, 8, b + 0),
            Slot(f"L{layer}.up", 4096, 14336, 8, b + 0),
            Slot(f"L{layer}.down", 14336, 4096, 8, b + 2))


def _llama_slots() -> Tuple[Slot, ...]:
    out: List[Slot] = []
    for l in range(32):
        b = 4 * l
        out += [Slot(f"L{l}.q", 4096, 4096, 1, b + 0),
                Slot(f"L{l}.k", 4096, 1024, 1, b + 0),
                Slot(f"L{l}.v", 4096, 1024, 1, b + 0),
                Slot(f"L{l}.o", 4096, 4096, 1, b + 3)]
    return tuple(out)


CONFIGS: Dict[str, Config] = {
    "tiny": Config("tiny", 1, (Slot("moe", 256, 256, 2, 0),), rank=8, n_adapters=4,
                   n_experts=2, top_k=1, n_tokens=64, y_dtype="fp32", no_lora_frac=0.1),
    "tiny_dense": Config("tiny_dense", 6, (Slot("dense", 256, 256, 1, 0),), rank=8, n_adapters=4,
                         n_experts=1, top_k=1, n_tokens=64, y_dtype="fp32", no_lora_frac=0.1),
    "llama_decode": Config("llama_decode", 2, _llama_slots(), rank=16, n_adapters=128,
                           n_experts=1, top_k=1, n_tokens=256, y_dtype="bf16"),
    "mixtral_decode": Config("mixtral_decode", 3, _moe_slots(), rank=64, n_adapters=512,
                             n_experts=8, top_k=2, n_tokens=512, y_dtype="bf16"),
    "mixtral_prefill": Config("mixtral_prefill", 4, _moe_slots(), rank=64, n_adapters=64,
                              n_experts=8, top_k=2, n_tokens=8192, y_dtype="bf16", n_seqs=4),
    "mixtral_sharded": Config("mixtral_sharded", 5, _moe_slots(), rank=64, n_adapters=2048,
                              n_experts=8, top_k=2, n_tokens=4096, y_dtype="bf16"),
}


# SURVEY 8d variants of the configs: uniform adapter ids (3u; Llama ~110
# distinct adapters) and the 16 x 512-token prefill (~77 units of 106-633 rows)
VARIANTS: Dict[str, Config] = {
    "mixtral_decode_uniform": dataclasses.replace(CONFIGS["mixtral_decode"], name="mixtral_decode_uniform",
                                                  zipf_s=0.0),
    "llama_decode_uniform": dataclasses.replace(CONFIGS["llama_decode"], name="llama_decode_uniform", zipf_s=0.0),
    "mixtral_prefill_16x512": dataclasses.replace(CONFIGS["mixtral_prefill"], name="mixtral_prefill_16x512",
                                                  n_seqs=16),
}


def with_tokens(cfg: Config, n_tokens: int, **kw) -> Config:
    """Same config at another batch size (parity sizes, batch sweeps)."""
    d = dataclasses.asdict(cfg)
    d["slots"] = cfg.slots
    d["n_tokens"] = n_tokens
    d.update(kw)
    return Config(**d)


# ----------------------------------------------------------------------------
# ids
# ----------------------------------------------------------------------------
def zipf_probs(n: int, s: float = 1.2) -> np.ndarray:
    """p_i proportional to i^-s over 1-based ranks; adapter id = rank - 1."""
    ranks = np.arange(1, n + 1, dtype=np.float64)
    w = ranks ** (-s)
    return w / w.sum()


@dataclasses.dataclass
class Batch:
    adapter_ids: np.ndarray   # int32 [T] per row (-1 = no LoRA)
    expert_ids: np.ndarray    # int32 [T] per row
    n_tokens: int
    top_k: int

    @property
    def n_rows(self) -> int:
        return int(self.adapter_ids.shape[0])


def make_batch(cfg: Config, seed: Optional[int] = None, skewed_experts: bool = False) -> Batch:
    """Per-row (adapter, expert) tags.  Rows are token-major: row t*k + j."""
    rng = np.random.Generator(np.random.PCG64(cfg.index if seed is None else seed))
    T, k, E = cfg.n_tokens, cfg.top_k, cfg.n_experts
    p = zipf_probs(cfg.n_adapters, cfg.zipf_s)
    if cfg.n_seqs > 0:
        seq_ad = rng.choice(cfg.n_adapters, size=cfg.n_seqs, p=p).astype(np.int32)
        per_seq = T // cfg.n_seqs
        tok_ad = np.repeat(seq_ad, per_seq)
        tok_ad = np.concatenate([tok_ad, np.full(T - tok_ad.size, seq_ad[-1], np.int32)])
    else:
        tok_ad = rng.choice(cfg.n_adapters, size=T, p=p).astype(np.int32)
    if cfg.no_lora_frac > 0:
        tok_ad = np.where(rng.random(T) < cfg.no_lora_frac, np.int32(-1), tok_ad).astype(np.int32)
    if E == 1:
        tok_ex = np.zeros((T, k), np.int32)
    else:
        if skewed_experts:
            w = zipf_probs(E, 1.0)
            keys = rng.random((T, E)) ** (1.0 / w)          # weighted sampling w/o replacement
            tok_ex = np.argsort(-keys, axis=1)[:, :k].astype(np.int32)
        else:
            tok_ex = np.argsort(rng.random((T, E)), axis=1)[:, :k].astype(np.int32)
    adapter_ids = np.repeat(tok_ad, k).astype(np.int32)
    expert_ids = tok_ex.reshape(-1).astype(np.int32)
    return Batch(adapter_ids, expert_ids, T, k)


def distinct_units(batch: Batch, E: int) -> int:
    v = batch.adapter_ids >= 0
    return int(np.unique(batch.adapter_ids[v].astype(np.int64) * E + batch.expert_ids[v]).size)


# ----------------------------------------------------------------------------
# full-mantissa inputs (x ~ N(0,1), A ~ N(0,1/h_in), B ~ N(0,1/r),
# y0 ~ N(0,1), rounded to bf16).  The counter-hash values above carry at most
# 8 significant bits; these exercise every mantissa bit and a wide exponent
# range.  Drawn with numpy PCG64; the fp32 -> bf16 step is round-to-nearest-
# even on the bit pattern (input preparation, not the method's arithmetic).
# ----------------------------------------------------------------------------
def f32_to_bf16_bits_rne(f: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return (u >> np.uint64(16)).astype(np.uint16)


def normal_bf16_bits(rng: np.random.Generator, shape, std: float = 1.0) -> np.ndarray:
    """bf16 bits of N(0, std^2) samples (finite, full mantissa)."""
    return f32_to_bf16_bits_rne((rng.standard_normal(shape) * std).astype(np.float32))
