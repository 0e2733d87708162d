"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars: segment/permutation indices bit-exact; exact-integer
probes bit-exact on every kernel path; floating point within
max|err| <= 1e-2*max|y| + 1e-3 (north_star), per slot; invariants bit-exact.
Small sizes compare every element; BASELINE.json's full sizes compare sampled
rows (the oracle computes them one by one), in the launch configuration that
bench.py times (multi-slot apply over one plan).
"""
import dataclasses

import numpy as np
import pytest
import torch

import lora_inputs as li
import oracle
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

from tests import gpu_util as U  # noqa: E402


@pytest.fixture(scope="module")
def B():
    return U.binding()


# ---------------------------------------------------------------------------
# a1 segmentation: bit-exact
# ---------------------------------------------------------------------------
def _plan_indices(B, s, ad, ex, T, E, max_rows):
    p = B.lora_plan_create(s, max_rows)
    try:
        B.lora_plan_build(s, p, ad, ex, T, E)
        perm = torch.empty(max_rows, dtype=torch.int32, device=U.DEV)
        off = torch.empty(max_rows + 1, dtype=torch.int32, device=U.DEV)
        keys = torch.empty(max_rows, dtype=torch.int32, device=U.DEV)
        nv, ns = B.lora_plan_export(s, p, perm, off, keys)
        return perm[:nv].cpu().numpy(), off[:ns + 1].cpu().numpy(), keys[:ns].cpu().numpy()
    finally:
        B.lora_plan_destroy(p)


@pytest.mark.parametrize("name", ["tiny", "tiny_dense", "llama_decode", "mixtral_decode", "mixtral_prefill",
                                  "mixtral_sharded"])
def test_segment_bit_exact_configs(B, name):
    cfg = li.CONFIGS[name]
    b = li.make_batch(cfg)
    # weights are irrelevant to a1: a small store with the config's adapter/expert space
    seg_cfg = li.Config(cfg.name, cfg.index, (li.Slot("s", 64, 64, cfg.n_experts, 0),), 8, cfg.n_adapters,
                        cfg.n_experts, cfg.top_k, cfg.n_tokens, "fp32")
    s = U.make_server(B, seg_cfg, max_rows=max(b.n_rows, 1), fill=False)
    try:
        ad, ex = U.ids_dev(b)
        perm, off, keys = _plan_indices(B, s, ad, ex, b.n_rows, cfg.n_experts, b.n_rows)
        rp, ro, rk = oracle.segment(b.adapter_ids, b.expert_ids, cfg.n_experts)
        np.testing.assert_array_equal(perm, rp)
        np.testing.assert_array_equal(off, ro)
        np.testing.assert_array_equal(keys, rk)
    finally:
        B.lora_server_destroy(s)


ADVERSARIAL = {
    "all_dropped": lambda rng: (np.full(100, -1), np.zeros(100)),
    "empty": lambda rng: (np.zeros(0), np.zeros(0)),
    "single": lambda rng: (np.array([37]), np.array([3])),
    "one_key": lambda rng: (np.full(5000, 7), np.full(5000, 2)),
    "all_distinct": lambda rng: (rng.permutation(4096), np.zeros(4096)),
    "top_of_range": lambda rng: (np.full(300, 4095), np.full(300, 3)),
    "max_rows_random": lambda rng: (rng.integers(-1, 4096, 16384), rng.integers(0, 4, 16384)),
    "ragged_1023": lambda rng: (rng.integers(-1, 50, 1023), rng.integers(0, 4, 1023)),
}


@pytest.mark.parametrize("case", sorted(ADVERSARIAL))
def test_segment_bit_exact_adversarial(B, case):
    rng = np.random.default_rng(11)
    a, e = ADVERSARIAL[case](rng)
    a, e = a.astype(np.int32), e.astype(np.int32)
    E = 4
    cfg = li.Config("adv", 9, (li.Slot("s", 64, 64, E, 0),), 8, 4096, E, 1, max(len(a), 1), "fp32")
    s = U.make_server(B, cfg, max_rows=16384, fill=False)
    try:
        ad = torch.from_numpy(a).to(U.DEV)
        ex = torch.from_numpy(e).to(U.DEV)
        perm, off, keys = _plan_indices(B, s, ad, ex, len(a), E, 16384)
        rp, ro, rk = oracle.segment(a, e, E)
        np.testing.assert_array_equal(perm, rp)
        np.testing.assert_array_equal(off, ro)
        np.testing.assert_array_equal(keys, rk)
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("T,n_ad,E", [(1, 16, 1), (1023, 64, 8), (2049, 16, 1), (4097, 2048, 8), (5000, 7, 3),
                                      (8192, 2048, 8), (16384, 64, 8), (16384, 4096, 4),
                                      (16385, 64, 8), (24000, 7, 3), (32768, 2048, 8)])
@pytest.mark.parametrize("multi", ["1", "0"])
def test_segment_multi_cta_path(B, monkeypatch, T, n_ad, E, multi):
    """Both segmenter paths (LORA_SEG_MULTI test hook: 1 = the multi-CTA
    local-sort / scan / scatter kernels at any T, 0 = the one-CTA kernel) give
    the oracle's stable segmentation bit-exactly, incl. -1 rows, Zipf-skewed
    and ragged batches, and a key space that makes the histogram wide.
    Above 16384 rows (one CTA's capacity) the multi-CTA path runs whatever the
    hook says (plan capacity 32768 rows)."""
    monkeypatch.setenv("LORA_SEG_MULTI", multi)
    rng = np.random.default_rng(T + n_ad)
    zipf = rng.choice(n_ad, size=T, p=li.zipf_probs(n_ad))
    a = np.where(rng.random(T) < 0.1, -1, zipf).astype(np.int32)
    e = rng.integers(0, E, T).astype(np.int32)
    cfg = li.Config("seg", 9, (li.Slot("s", 64, 64, E, 0),), 8, n_ad, E, 1, T, "fp32")
    s = U.make_server(B, cfg, max_rows=T, fill=False)
    p = B.lora_plan_create(s, T)
    try:
        # a first build on other ids: the second must not see its histogram
        a0 = torch.from_numpy(rng.integers(0, n_ad, T).astype(np.int32)).to(U.DEV)
        B.lora_plan_build(s, p, a0, None if E == 1 else torch.zeros(T, dtype=torch.int32, device=U.DEV), T, E)
        B.lora_plan_build(s, p, torch.from_numpy(a).to(U.DEV), torch.from_numpy(e).to(U.DEV) if E > 1 else None,
                          T, E)
        perm = torch.empty(T, dtype=torch.int32, device=U.DEV)
        off = torch.empty(T + 1, dtype=torch.int32, device=U.DEV)
        keys = torch.empty(T, dtype=torch.int32, device=U.DEV)
        nv, ns = B.lora_plan_export(s, p, perm, off, keys)
        rp, ro, rk = oracle.segment(a, e if E > 1 else None, E)
        np.testing.assert_array_equal(perm[:nv].cpu().numpy(), rp)
        np.testing.assert_array_equal(off[:ns + 1].cpu().numpy(), ro)
        np.testing.assert_array_equal(keys[:ns].cpu().numpy(), rk)
    finally:
        B.lora_plan_destroy(p)
        B.lora_server_destroy(s)


# ---------------------------------------------------------------------------
# generator identity (the CUDA fill implements the same recipe)
# ---------------------------------------------------------------------------
def test_fill_rows_matches_generator(B):
    x = torch.empty((37, 320), dtype=torch.int16, device=U.DEV)
    B.lora_synth_fill_rows(x, 37, 320, 1234, li.tag_of(li.KIND_X, 5), li.shift_x(), 1000)
    ref = li.x_rows_bits(1234, 5, np.arange(1000, 1037), 320)
    np.testing.assert_array_equal(x.cpu().numpy().view(np.uint16), ref)


@pytest.mark.parametrize("rank", [8, 16, 32, 64, 128])
def test_fill_store_equals_loaded_weights(B, rank):
    """Server filled on device == server loaded from numpy-generated weights (bit-exact y)."""
    E, n_ad, h_in, h_out, T = 2, 3, 128, 192, 40
    cfg = li.Config("fill", 7, (li.Slot("s", h_in, h_out, E, 0),), rank, n_ad, E, 1, T, "fp32")
    A = np.stack([li.unit_A_bits(cfg.seed, 0, u, h_in, rank) for u in range(n_ad * E)])
    Bw = np.stack([li.unit_B_bits(cfg.seed, 0, u, rank, h_out) for u in range(n_ad * E)])
    c = B.make_config([h_in], [h_out], [E], rank, n_ad, cfg.scale(), T, 0)
    s1 = B.lora_server_create(c, [A], [Bw], weights_on_device=False)
    s2 = U.make_server(B, cfg)
    try:
        rng = np.random.default_rng(1)
        a = torch.from_numpy(rng.integers(-1, n_ad, T).astype(np.int32)).to(U.DEV)
        e = torch.from_numpy(rng.integers(0, E, T).astype(np.int32)).to(U.DEV)
        x = U.x_dev(B, cfg, 0, T)
        y1 = U.y0_dev(B, cfg, 0, T)
        y2 = y1.clone()
        B.lora_apply(s1, 0, x, a, e, y1, B.LORA_FP32, T)
        B.lora_apply(s2, 0, x, a, e, y2, B.LORA_FP32, T)
        torch.cuda.synchronize()
        assert torch.equal(y1.view(torch.int32), y2.view(torch.int32))
    finally:
        B.lora_server_destroy(s1)
        B.lora_server_destroy(s2)


# ---------------------------------------------------------------------------
# exact-integer probes: bit-exact on every kernel path
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("rank,small_max", [(8, None), (16, None), (32, None), (64, -1), (64, 0), (64, 4),
                                            (128, None), (16, 0), (16, 4), (32, 0), (32, 4), (128, 0), (128, 4),
                                            (8, 0), (8, 4)])
def test_exact_integer_probes(B, monkeypatch, rank, small_max):
    """Every kernel route bit-exact on integer-valued inputs: CUDA cores only
    (small_max -1), tcgen05 only (small_max 0), or both (the large segment on
    tcgen05 at r = 8 / 16 / 32 / 64 / 128, LORA_TC_MIN_ROWS=0)."""
    if rank != 64 and small_max is not None:
        monkeypatch.setenv("LORA_TC_MIN_ROWS", "0")
    rng = np.random.default_rng(rank * 10 + (3 if small_max is None else small_max + 2))
    E, n_ad, h_in, h_out, T = 2, 40, 128, 256, 300   # widths multiple of 128: tcgen05-eligible
    Ai = rng.integers(-1, 2, (n_ad * E, h_in, rank))
    Bi = rng.integers(-1, 2, (n_ad * E, rank, h_out))
    xi = rng.integers(-2, 3, (T, h_in))
    yi = rng.integers(-50, 51, (T, h_out)).astype(np.float32)
    a = rng.integers(-1, n_ad, T).astype(np.int32)
    a[:120] = 1                      # one large segment (tcgen05 path when enabled)
    e = rng.integers(0, E, T).astype(np.int32)
    scale = np.array([(0.5, 1.0, 2.0)[i % 3] for i in range(n_ad)], np.float32)
    bits = lambda v: li.f32_to_bf16_bits_exact(np.asarray(v, np.float32))
    c = B.make_config([h_in], [h_out], [E], rank, n_ad, scale, T, 0)
    s = B.lora_server_create(c, [bits(Ai)], [bits(Bi)], weights_on_device=False)
    try:
        if small_max is not None:
            B.lora_server_set_small_seg_max(s, small_max)
        x = torch.from_numpy(bits(xi).view(np.int16)).to(U.DEV)
        y = torch.from_numpy(yi.copy()).to(U.DEV)
        p = B.lora_plan_create(s, T)
        B.lora_plan_build(s, p, torch.from_numpy(a).to(U.DEV), torch.from_numpy(e).to(U.DEV), T, E)
        nv, ns, ng, nt = B.lora_plan_stats(s, p)
        # the requested kernel path is the one that ran
        # (conftest sets LORA_TC_MIN_ROWS=0: the large segment takes tcgen05 at every tcgen05 rank)
        if small_max == -1:
            assert nt == 0 and ng > 0
        elif small_max == 0:
            assert ng == 0 and nt > 0
        else:
            assert ng > 0 and nt > 0
        B.lora_apply_plan(s, p, 0, x, y, B.LORA_FP32)
        torch.cuda.synchronize()
        B.lora_plan_destroy(p)
        exp = yi.astype(np.float64).copy()
        for i in range(T):
            if a[i] >= 0:
                u = a[i] * E + e[i]
                exp[i] += float(scale[a[i]]) * ((xi[i] @ Ai[u]) @ Bi[u])
        np.testing.assert_array_equal(y.cpu().numpy(), exp.astype(np.float32))
    finally:
        B.lora_server_destroy(s)


# ---------------------------------------------------------------------------
# float parity against the oracle
# ---------------------------------------------------------------------------
def _run_multi(B, s, cfg, batch, slot_ids, y0="random", host=False):
    T = batch.n_rows
    ad, ex = U.ids_dev(batch)
    E = cfg.slots[slot_ids[0]].n_experts
    xs = {}
    for i in slot_ids:
        xb = cfg.slots[i].xbuf
        if xb not in xs:
            xs[xb] = U.x_dev(B, cfg, i, T)
    ys = [U.y0_dev(B, cfg, i, T, y0) for i in slot_ids]
    dt = B.LORA_FP32 if cfg.y_dtype == "fp32" else B.LORA_BF16
    p = B.lora_plan_create(s, T)
    try:
        B.lora_plan_build(s, p, ad, ex if E > 1 else None, T, E)
        B.lora_apply_plan_multi(s, p, list(slot_ids), [xs[cfg.slots[i].xbuf] for i in slot_ids], ys, dt)
        torch.cuda.synchronize()
        assert B.lora_server_check(s) == B.LORA_OK
    finally:
        B.lora_plan_destroy(p)
    return ys


def _run_multi_unchecked(B, s, cfg, batch, slot_ids):
    """_run_multi without asserting a clean sticky flag (rows may be rejected)."""
    T = batch.n_rows
    ad, ex = U.ids_dev(batch)
    E = cfg.slots[slot_ids[0]].n_experts
    xs = {}
    for i in slot_ids:
        if cfg.slots[i].xbuf not in xs:
            xs[cfg.slots[i].xbuf] = U.x_dev(B, cfg, i, T)
    ys = [U.y0_dev(B, cfg, i, T) for i in slot_ids]
    p = B.lora_plan_create(s, T)
    try:
        B.lora_plan_build(s, p, ad, ex if E > 1 else None, T, E)
        B.lora_apply_plan_multi(s, p, list(slot_ids), [xs[cfg.slots[i].xbuf] for i in slot_ids], ys,
                                B.LORA_FP32 if cfg.y_dtype == "fp32" else B.LORA_BF16)
        torch.cuda.synchronize()
    finally:
        B.lora_plan_destroy(p)
    return ys


@pytest.mark.parametrize("name,y0,small_max", [("tiny", "random", None), ("tiny", "zero", None),
                                                ("tiny_dense", "random", None), ("tiny", "random", -1)])
def test_tiny_all_elements(B, name, y0, small_max):
    cfg = li.CONFIGS[name]
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg, small_max=small_max)
    try:
        (y,) = _run_multi(B, s, cfg, b, [0], y0)
        ref = oracle.apply_slot(cfg, 0, b, y0=y0)
        U.assert_parity(y, ref, name)
        # rows with a = -1 untouched, bit-exact
        none = b.adapter_ids < 0
        if y0 == "random":
            y00 = U.y0_dev(B, cfg, 0, b.n_rows, y0)
            assert torch.equal(y[torch.from_numpy(none).to(U.DEV)].view(torch.int32),
                               y00[torch.from_numpy(none).to(U.DEV)].view(torch.int32))
    finally:
        B.lora_server_destroy(s)


def test_llama_decode_two_layers_all_rows(B):
    cfg = li.CONFIGS["llama_decode"]
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg, n_slots=8)
    try:
        ys = _run_multi(B, s, cfg, b, list(range(8)))
        for i in range(8):
            ref = oracle.apply_slot(cfg, i, b, n_threads=0)
            U.assert_parity(ys[i], ref, f"llama slot {i}")
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("name,small_max", [("mixtral_decode", None), ("mixtral_decode", -1),
                                            ("mixtral_prefill", None)])
def test_mixtral_sampled_rows(B, name, small_max):
    cfg = li.CONFIGS[name]
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg, small_max=small_max)
    try:
        ys = _run_multi(B, s, cfg, b, [0, 1, 2])
        rows = U.sample_rows(b, 40, E=cfg.n_experts)
        for i in range(3):
            ref = oracle.apply_slot(cfg, i, b, rows=rows)
            U.assert_parity(ys[i][torch.from_numpy(rows).to(U.DEV)], ref, f"{name} slot {i}")
    finally:
        B.lora_server_destroy(s)


@pytest.mark.slow
def test_mixtral_sharded_config_at_g1_sampled(B):
    """Config 5 on one GPU (116 GB of weights), the bench's N=1 workload."""
    cfg = li.CONFIGS["mixtral_sharded"]
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        ys = _run_multi(B, s, cfg, b, [0, 1, 2])
        rows = U.sample_rows(b, 24, E=cfg.n_experts)
        for i in range(3):
            ref = oracle.apply_slot(cfg, i, b, rows=rows)
            U.assert_parity(ys[i][torch.from_numpy(rows).to(U.DEV)], ref, f"sharded-g1 slot {i}")
    finally:
        B.lora_server_destroy(s)


@pytest.mark.slow
def test_mixtral_sharded_config_push_loopback_sampled(B, monkeypatch):
    """Config 5 at full size through the sharded server's push path
    (loopback: every row goes through bucket / announce / recv-prep, the
    owner's shrink reads x rows through the registered mapping, the expand
    epilogue red.adds the deltas into the registered y)."""
    monkeypatch.setenv("LORA_SHARD_LOOPBACK", "1")
    cfg = li.CONFIGS["mixtral_sharded"]
    b = li.make_batch(cfg)
    T = b.n_rows
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                      [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(), T, 0)
    sh = B.lora_server_create_sharded(c, 0, 1, B.lora_nccl_unique_id())
    try:
        B.lora_server_fill_synthetic(sh, cfg.seed)
        ad, ex = U.ids_dev(b)
        xs = {}
        for i, sl in enumerate(cfg.slots):
            if sl.xbuf not in xs:
                xs[sl.xbuf] = U.x_dev(B, cfg, i, T)
        ys = [U.y0_dev(B, cfg, i, T) for i in range(3)]
        U.register(B, sh, list(xs.values()) + ys)
        B.lora_apply_sharded(sh, [0, 1, 2], [xs[sl.xbuf] for sl in cfg.slots], ad, ex, ys, B.LORA_BF16, T)
        torch.cuda.synchronize()
        assert B.lora_server_check(sh) == B.LORA_OK
        rows = U.sample_rows(b, 24, E=cfg.n_experts)
        for i in range(3):
            ref = oracle.apply_slot(cfg, i, b, rows=rows)
            U.assert_parity(ys[i][torch.from_numpy(rows).to(U.DEV)], ref, f"push loopback slot {i}")
    finally:
        B.lora_server_destroy(sh)


# ---------------------------------------------------------------------------
# invariants and API equivalences (bit-exact)
# ---------------------------------------------------------------------------
def _mid_cfg(rank=64, T=600):
    return li.Config("mid", 8, (li.Slot("a", 512, 768, 4, 0), li.Slot("b", 768, 512, 4, 1)), rank, 24, 4, 2,
                     T // 2, "bf16")


def test_determinism_and_multi_equals_single(B):
    cfg = _mid_cfg()
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        y_multi = _run_multi(B, s, cfg, b, [0, 1])
        y_again = _run_multi(B, s, cfg, b, [0, 1])
        for u, v in zip(y_multi, y_again):
            assert torch.equal(u, v)
        for i in range(2):
            (y1,) = _run_multi(B, s, cfg, b, [i])
            assert torch.equal(y1, y_multi[i])
            ref = oracle.apply_slot(cfg, i, b)
            U.assert_parity(y1, ref, f"mid slot {i}")
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("case", ["single_row", "one_segment", "all_no_lora", "ragged_mixed"])
def test_edge_cases(B, case):
    """Degenerate batches: one row; one (adapter, expert) unit holding every
    row (one segment -> tcgen05 tiles with a near-equal split); no row with a
    LoRA (y untouched, bit-exact); an odd row count mixing -1 rows, every
    element checked against the oracle."""
    T = {"single_row": 1, "one_segment": 300, "all_no_lora": 64, "ragged_mixed": 257}[case]
    cfg = dataclasses.replace(_mid_cfg(), top_k=1, n_tokens=T)
    r = np.arange(T)
    if case == "single_row":
        a, e = np.array([3]), np.array([1])
    elif case == "one_segment":
        a, e = np.full(T, 7), np.full(T, 2)
    elif case == "all_no_lora":
        a, e = np.full(T, -1), np.zeros(T)
    else:
        a, e = (r % 3) - 1, r % 4
    b = li.Batch(a.astype(np.int32), e.astype(np.int32), T, 1)
    s = U.make_server(B, cfg)
    try:
        y0 = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        ys = _run_multi(B, s, cfg, b, [0, 1])
        for i in range(2):
            if case == "all_no_lora":
                assert torch.equal(ys[i], y0[i])
            else:
                U.assert_parity(ys[i], oracle.apply_slot(cfg, i, b), f"{case} slot {i}")
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("rank", [8, 16, 64, 128])
def test_resident_cache_matches_full_store(B, rank):
    """Resident-adapter cache (n_resident = 6 of 24 adapters, weights in
    pinned host memory, lora_server_require with LRU eviction and per-slot
    copies): bit-identical to the fully resident server on batches drawn from
    changing adapter subsets; a repeated subset copies nothing; a row whose
    adapter is not resident is skipped and flagged."""
    cfg = _mid_cfg(rank=rank, T=400)
    full = U.make_server(B, cfg)
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                      [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(), 400, 0,
                      n_resident=6)
    cs = B.lora_server_create(c)
    try:
        B.lora_server_fill_synthetic(cs, cfg.seed)
        rng = np.random.default_rng(11)
        T = 400
        subsets = [[0, 1, 2, 3], [0, 1, 2, 3], [4, 5, 6, 7, 8, 9], [0, 5, 23, 12], [12, 13, 14, 15, 16, 17]]
        expect_loads = [4, 0, 6, None, None]
        for it, sub in enumerate(subsets):
            a = rng.choice(np.array(sub + [-1]), T).astype(np.int32)
            e = rng.integers(0, cfg.n_experts, T).astype(np.int32)
            b = li.Batch(a, e, T, 1)
            loaded = B.lora_server_require(cs, sub)
            if expect_loads[it] is not None:
                assert loaded == expect_loads[it], (it, loaded)
            y_full = _run_multi(B, full, cfg, b, [0, 1])
            y_cache = _run_multi(B, cs, cfg, b, [0, 1])
            for i in range(2):
                assert torch.equal(y_cache[i], y_full[i]), (it, i)
        # adapter 20 is not resident: its rows are skipped and flagged
        a = np.full(T, 12, np.int32)
        a[5] = 20
        b = li.Batch(a, np.zeros(T, np.int32), T, 1)
        y0 = U.y0_dev(B, cfg, 0, T)
        x = U.x_dev(B, cfg, 0, T)
        ad = torch.from_numpy(a).to(U.DEV)
        ex = torch.zeros(T, dtype=torch.int32, device=U.DEV)
        y = y0.clone()
        B.lora_apply(cs, 0, x, ad, ex, y, B.LORA_BF16, T)
        assert B.lora_server_check(cs) == B.LORA_ERR_ID_OUT_OF_RANGE
        assert torch.equal(y[5], y0[5])
    finally:
        B.lora_server_destroy(cs)
        B.lora_server_destroy(full)


@pytest.mark.parametrize("world,rank,ep,n_hot", [(2, 0, 0, 0), (2, 1, 0, 0), (3, 2, 0, 4), (2, 1, 1, 0), (3, 1, 1, 0)])
def test_sharded_store_layouts_fake_world(B, monkeypatch, world, rank, ep, n_hot):
    """The store of one rank of a sharded server (LORA_FAKE_WORLD test hook:
    same placement, no communicator) for LoRA Data Parallel striping, with
    replicated hot adapters, and expert parallel: rows of the units that rank
    owns match the oracle, every other row is skipped (y untouched) and
    flagged."""
    monkeypatch.setenv("LORA_FAKE_WORLD", f"{world},{rank},{ep},{n_hot}")
    cfg = _mid_cfg(T=500)
    b = li.make_batch(cfg)
    T = b.n_rows
    s = U.make_server(B, cfg)
    try:
        src = np.full(T, rank)
        own = orc.owner_of(b.adapter_ids, world, n_hot, src, b.expert_ids, bool(ep))
        mine = own == rank
        y0 = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        ys = _run_multi_unchecked(B, s, cfg, b, [0, 1])
        assert B.lora_server_check(s) == (B.LORA_ERR_ID_OUT_OF_RANGE if np.any(own >= 0) and not np.all(mine | (own < 0)) else B.LORA_OK)
        rows = np.flatnonzero(mine)
        assert rows.size > 0
        other = torch.from_numpy(np.flatnonzero(~mine)).to(U.DEV)
        for i in range(2):
            ref = oracle.apply_slot(cfg, i, b, rows=rows)
            U.assert_parity(ys[i][torch.from_numpy(rows).to(U.DEV)], ref, f"fake world slot {i}")
            assert torch.equal(ys[i][other], y0[i][other])
    finally:
        B.lora_server_destroy(s)


def test_cuda_graph_replay_bit_exact(B):
    """A step (plan build + multi-slot apply, including the fork/join of the
    tcgen05 side stream) captured in a CUDA graph and replayed gives the
    eager result bit for bit (bench.py times the replay)."""
    cfg = _mid_cfg()
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        T = b.n_rows
        y_eager = _run_multi(B, s, cfg, b, [0, 1])
        ad, ex = U.ids_dev(b)
        xs = [U.x_dev(B, cfg, i, T) for i in range(2)]
        ys = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        y_init = [y.clone() for y in ys]
        p = B.lora_plan_create(s, T)
        g_stream = torch.cuda.Stream()
        g_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(g_stream):
            B.lora_plan_build(s, p, ad, ex, T, cfg.n_experts, g_stream)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=g_stream):
                B.lora_plan_build(s, p, ad, ex, T, cfg.n_experts, g_stream)
                B.lora_apply_plan_multi(s, p, [0, 1], xs, ys, B.LORA_BF16, g_stream)
        torch.cuda.current_stream().wait_stream(g_stream)
        for y, y0 in zip(ys, y_init):
            y.copy_(y0)
        graph.replay()
        torch.cuda.synchronize()
        for i in range(2):
            assert torch.equal(ys[i], y_eager[i])
        B.lora_plan_destroy(p)
    finally:
        B.lora_server_destroy(s)


def test_permutation_equivariance_bit_exact(B):
    cfg = _mid_cfg()
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        T = b.n_rows
        (y,) = _run_multi(B, s, cfg, b, [0])
        perm = np.random.default_rng(3).permutation(T)
        ad = torch.from_numpy(b.adapter_ids[perm]).to(U.DEV)
        ex = torch.from_numpy(b.expert_ids[perm]).to(U.DEV)
        pt = torch.from_numpy(perm).to(U.DEV)
        x = U.x_dev(B, cfg, 0, T)[pt].contiguous()
        yp = U.y0_dev(B, cfg, 0, T)[pt].contiguous()
        B.lora_apply(s, 0, x, ad, ex, yp, B.LORA_BF16, T)
        torch.cuda.synchronize()
        assert torch.equal(yp, y[pt])
    finally:
        B.lora_server_destroy(s)


def test_host_entry_equals_device_path(B):
    cfg = _mid_cfg()
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        T = b.n_rows
        y_dev = _run_multi(B, s, cfg, b, [0, 1])
        xh = [U.x_dev(B, cfg, i, T).cpu().pin_memory() for i in range(2)]
        yh = [U.y0_dev(B, cfg, i, T).cpu().pin_memory() for i in range(2)]
        B.lora_apply_multi_host(s, [0, 1], xh, b.adapter_ids, b.expert_ids, yh, B.LORA_BF16, T)
        torch.cuda.synchronize()
        for i in range(2):
            assert torch.equal(yh[i], y_dev[i].cpu())
    finally:
        B.lora_server_destroy(s)


def test_out_of_range_ids_flagged_and_skipped(B):
    cfg = _mid_cfg(T=64)
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        T = b.n_rows
        a = b.adapter_ids.copy()
        a[3] = cfg.n_adapters + 5
        e = b.expert_ids.copy()
        e[7] = 9
        x = U.x_dev(B, cfg, 0, T)
        y = U.y0_dev(B, cfg, 0, T)
        y0 = y.clone()
        B.lora_apply(s, 0, x, torch.from_numpy(a).to(U.DEV), torch.from_numpy(e).to(U.DEV), y, B.LORA_BF16, T)
        assert B.lora_server_check(s) == B.LORA_ERR_ID_OUT_OF_RANGE
        assert B.lora_server_check(s) == B.LORA_OK        # flag cleared
        assert torch.equal(y[3], y0[3]) and torch.equal(y[7], y0[7])
    finally:
        B.lora_server_destroy(s)


def test_argument_errors_enqueue_nothing(B):
    cfg = _mid_cfg(T=64)
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        T = b.n_rows
        ad, ex = U.ids_dev(b)
        x = U.x_dev(B, cfg, 0, T)
        y = U.y0_dev(B, cfg, 0, T)
        y0 = y.clone()
        with pytest.raises(B.LoraError) as ei:
            B.lora_apply(s, 5, x, ad, ex, y, B.LORA_BF16, T)
        assert ei.value.status == B.LORA_ERR_INVALID_ARG
        with pytest.raises(B.LoraError):
            B.lora_apply(s, 0, x, ad, ex, y, B.LORA_BF16, 10 ** 6)
        p = B.lora_plan_create(s, T)
        B.lora_plan_build(s, p, ad, ex, T, 2)          # E mismatch with the slot (E=4)
        with pytest.raises(B.LoraError):
            B.lora_apply_plan(s, p, 0, x, y, B.LORA_BF16)
        with pytest.raises(B.LoraError):                 # x / y overlap
            B.lora_apply_plan_multi(s, p, [0], [y], [y], B.LORA_BF16)
        B.lora_plan_destroy(p)
        B.lora_apply(s, 0, x, ad, ex, y, B.LORA_BF16, 0)  # T = 0: no-op
        torch.cuda.synchronize()
        assert torch.equal(y, y0)
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("rank", [8, 16, 32])
def test_small_rank_bf16_full_parity(B, rank):
    """r <= 32 takes the CUDA-core path with two columns per thread and the
    smem-tile + bulk-store output (bf16 y); every element checked."""
    cfg = _mid_cfg(rank=rank)
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        ys = _run_multi(B, s, cfg, b, [0, 1])
        for i in range(2):
            U.assert_parity(ys[i], oracle.apply_slot(cfg, i, b), f"r={rank} slot {i}")
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("y_dtype", ["bf16", "fp32"])
def test_beyond_one_cta_rows_full_parity(B, y_dtype):
    """A 20000-row batch (above the one-CTA segmenter's 16384; plan capacity
    32768): multi-CTA segmenter, tcgen05 whole-K tiles beside CUDA-core
    groups; every element against the oracle."""
    cfg = dataclasses.replace(_mid_cfg(rank=64, T=20000), y_dtype=y_dtype)
    b = li.make_batch(cfg)
    assert b.n_rows == 20000
    s = U.make_server(B, cfg)
    try:
        ys = _run_multi(B, s, cfg, b, [0, 1])
        for i in range(2):
            U.assert_parity(ys[i], oracle.apply_slot(cfg, i, b), f"20000 rows {y_dtype} slot {i}")
    finally:
        B.lora_server_destroy(s)


def test_plan_capacity_bound(B):
    """max_rows 32768 is accepted, 32769 rejected (LORA_ERR_UNSUPPORTED)."""
    cfg = _mid_cfg(rank=16, T=600)
    s = U.make_server(B, cfg, fill=False)
    try:
        p = B.lora_plan_create(s, 32768)
        B.lora_plan_destroy(p)
        with pytest.raises(B.LoraError) as ei:
            B.lora_plan_create(s, 32769)
        assert ei.value.status == B.LORA_ERR_UNSUPPORTED
    finally:
        B.lora_server_destroy(s)


def _tc_rank_cfg(rank, T, y_dtype):
    # slot c's h_in = 16384 splits K on the tcgen05 chain below 4096 rows at
    # every rank (KI caps 8192 / 4096 / 2048 / 512 at r = 8 / 16 / 32 / 128): tc_vreduce
    return li.Config("tcr", 12, (li.Slot("a", 512, 768, 4, 0), li.Slot("b", 768, 512, 4, 1),
                                 li.Slot("c", 16384, 256, 4, 2)), rank, 24, 4, 2, T // 2, y_dtype)


@pytest.mark.parametrize("rank", [8, 16, 32, 128])
@pytest.mark.parametrize("y_dtype,T,small_max", [("bf16", 600, None), ("fp32", 600, 0), ("bf16", 4200, None)])
def test_tc_chain_every_rank_full_parity(B, monkeypatch, rank, y_dtype, T, small_max):
    """The tcgen05 chain at r = 16 / 32 / 128 (SWIZZLE_32B / 64B v and Bt
    operands; r = 128: two K blocks, Bt rows re-tiled by the producer warp),
    forced on with LORA_TC_MIN_ROWS=0: K-split + tc_vreduce (T = 600) and
    whole-K (T = 4200 rows >= 4096) items, tcgen05 tiles beside CUDA-core
    groups (small_max None) or every row on tcgen05 (0); every element."""
    monkeypatch.setenv("LORA_TC_MIN_ROWS", "0")
    cfg = _tc_rank_cfg(rank, T, y_dtype)
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg, small_max=small_max)
    try:
        p = B.lora_plan_create(s, cfg.n_rows)
        ad, ex = U.ids_dev(b)
        B.lora_plan_build(s, p, ad, ex, cfg.n_rows, 4)
        nv, ns, ng, nt = B.lora_plan_stats(s, p)
        B.lora_plan_destroy(p)
        assert nt > 0, "the tcgen05 chain did not run"
        ys = _run_multi(B, s, cfg, b, [0, 1, 2])
        for i in range(3):
            U.assert_parity(ys[i], oracle.apply_slot(cfg, i, b), f"tc r={rank} {y_dtype} T={T} slot {i}")
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("y_dtype,T", [("bf16", 600), ("fp32", 600), ("bf16", 24), ("fp32", 4000)])
def test_rank128_full_parity(B, y_dtype, T):
    """r = 128 (the top of the paper's "r typically 32-128"): the
    mma.sync shrink with one 16-row M tile per consumer warp and the expand
    with two threads per output column; every element checked, with and
    without the device K-split (T = 24: few items, split; T = 4000: whole K)."""
    cfg = dataclasses.replace(_mid_cfg(rank=128, T=T), y_dtype=y_dtype)
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        ys = _run_multi(B, s, cfg, b, [0, 1])
        for i in range(2):
            U.assert_parity(ys[i], oracle.apply_slot(cfg, i, b), f"r=128 {y_dtype} T={T} slot {i}")
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("loopback,y_dtype,rank,transport", [
    (False, "bf16", 64, "push"), (True, "fp32", 64, "push"), (True, "bf16", 64, "push"), (True, "bf16", 16, "push"),
    (True, "fp32", 16, "push"), (True, "fp32", 8, "nccl"), (True, "bf16", 128, "push"), (True, "fp32", 128, "push"),
    (True, "fp32", 64, "nccl"), (True, "bf16", 64, "nccl"), (True, "bf16", 8, "push"), (True, "fp32", 32, "push")])
def test_sharded_g1(B, monkeypatch, loopback, y_dtype, rank, transport):
    """Sharded server at G = 1.  In place (no exchange): bit-identical to the
    unsharded server.  Loopback (LORA_SHARD_LOOPBACK=1 sends every row through
    the exchange to itself, so one GPU runs the whole sharded path) with
    either path: push (x / y registered: device-side counts, the owner's
    shrink reads x rows through the registered mapping, the expand epilogue
    red.adds the deltas into the registered y) or nccl (unregistered: grouped
    send/recv + scatter-add).  fp32 y: bit-identical to the unsharded server
    (R18); bf16 y returns bf16 deltas (R19) and is held to the oracle
    tolerance, every row.  Three calls: buffers and the epoch are reused."""
    cfg = dataclasses.replace(_mid_cfg(rank=rank), y_dtype=y_dtype)
    if loopback:
        monkeypatch.setenv("LORA_SHARD_LOOPBACK", "1")
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    T = b.n_rows
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                      [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(), T, 0)
    uid = B.lora_nccl_unique_id()
    sh = B.lora_server_create_sharded(c, 0, 1, uid)
    try:
        B.lora_server_fill_synthetic(sh, cfg.seed)
        y_ref = _run_multi(B, s, cfg, b, [0, 1])
        ad, ex = U.ids_dev(b)
        xs = [U.x_dev(B, cfg, i, T) for i in range(2)]
        y0 = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        ys = [v.clone() for v in y0]
        if transport == "push":
            U.register(B, sh, xs + ys)
        dt = B.LORA_FP32 if y_dtype == "fp32" else B.LORA_BF16
        for rep in range(3):
            for v, v0 in zip(ys, y0):
                v.copy_(v0)
            B.lora_apply_sharded(sh, [0, 1], xs, ad, ex, ys, dt, T)
            torch.cuda.synchronize()
            assert B.lora_server_check(sh) == B.LORA_OK
            for i in range(2):
                if loopback and y_dtype == "bf16":
                    U.assert_parity(ys[i], oracle.apply_slot(cfg, i, b), f"loopback bf16 slot {i}")
                else:
                    assert torch.equal(ys[i], y_ref[i]), f"slot {i} rep {rep}"
    finally:
        B.lora_server_destroy(sh)
        B.lora_server_destroy(s)


@pytest.mark.parametrize("y_dtype", ["fp32", "bf16"])
def test_sharded_loopback_beyond_one_cta_rows(B, monkeypatch, y_dtype):
    """A 20000-row batch through the push path's loopback: the owner-side plan
    (capacity max_rows * world, row count known on the device) takes the
    multi-CTA segmenter with the rows past the device count masked.  fp32:
    bit-identical to the unsharded server; bf16: the oracle's tolerance."""
    monkeypatch.setenv("LORA_SHARD_LOOPBACK", "1")
    cfg = dataclasses.replace(_mid_cfg(rank=64, T=20000), y_dtype=y_dtype)
    b = li.make_batch(cfg)
    T = b.n_rows
    s = U.make_server(B, cfg)
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                      [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(), T, 0)
    sh = B.lora_server_create_sharded(c, 0, 1, B.lora_nccl_unique_id())
    try:
        B.lora_server_fill_synthetic(sh, cfg.seed)
        y_ref = _run_multi(B, s, cfg, b, [0, 1])
        ad, ex = U.ids_dev(b)
        xs = [U.x_dev(B, cfg, i, T) for i in range(2)]
        ys = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        U.register(B, sh, xs + ys)
        B.lora_apply_sharded(sh, [0, 1], xs, ad, ex, ys, B.LORA_FP32 if y_dtype == "fp32" else B.LORA_BF16, T)
        torch.cuda.synchronize()
        assert B.lora_server_check(sh) == B.LORA_OK
        for i in range(2):
            if y_dtype == "fp32":
                assert torch.equal(ys[i], y_ref[i]), f"slot {i}"
            else:
                U.assert_parity(ys[i], oracle.apply_slot(cfg, i, b), f"loopback 20000 rows slot {i}")
    finally:
        B.lora_server_destroy(sh)
        B.lora_server_destroy(s)


def test_sharded_push_graph_capture(B, monkeypatch):
    """The push path has no host synchronisation: a sharded step captured in a
    CUDA graph and replayed (the epoch advances in device memory) gives the
    eager result bit for bit, replay after replay."""
    monkeypatch.setenv("LORA_SHARD_LOOPBACK", "1")
    cfg = dataclasses.replace(_mid_cfg(rank=64), y_dtype="fp32")
    b = li.make_batch(cfg)
    T = b.n_rows
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                      [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(), T, 0)
    sh = B.lora_server_create_sharded(c, 0, 1, B.lora_nccl_unique_id())
    s = U.make_server(B, cfg)
    try:
        B.lora_server_fill_synthetic(sh, cfg.seed)
        y_ref = _run_multi(B, s, cfg, b, [0, 1])
        ad, ex = U.ids_dev(b)
        xs = [U.x_dev(B, cfg, i, T) for i in range(2)]
        y0 = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        ys = [v.clone() for v in y0]
        U.register(B, sh, xs + ys)
        g_stream = torch.cuda.Stream()
        g_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(g_stream):
            B.lora_apply_sharded(sh, [0, 1], xs, ad, ex, ys, B.LORA_FP32, T, g_stream)  # warm-up (eager)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=g_stream):
                B.lora_apply_sharded(sh, [0, 1], xs, ad, ex, ys, B.LORA_FP32, T, g_stream)
        torch.cuda.current_stream().wait_stream(g_stream)
        torch.cuda.synchronize()
        for rep in range(3):
            for v, v0 in zip(ys, y0):
                v.copy_(v0)
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            assert B.lora_server_check(sh) == B.LORA_OK
            for i in range(2):
                assert torch.equal(ys[i], y_ref[i]), f"replay {rep} slot {i}"
    finally:
        B.lora_server_destroy(sh)
        B.lora_server_destroy(s)


@pytest.mark.parametrize("rank", [0, 1, 2, 3])
def test_hybrid_ep2_pp2_store_fake_world(B, monkeypatch, rank):
    """Hybrid EP_x-PP_y placement with x = 2, y = 2 on a world of
    4 (LORA_FAKE_WORLD test hook, fifth field = pp stages): layers 0 and 1
    (two slots each) interleave over the two groups (layer l -> ranks
    (l mod 2) * 2 + e mod 2).  This rank's own layer: the rows whose expert it
    owns match the oracle, the rest stay untouched and are flagged.  The
    other group's layer: the apply is rejected (no unit stored)."""
    monkeypatch.setenv("LORA_FAKE_WORLD", f"4,{rank},1,0,2")
    cfg = li.Config("hyb", 8, (li.Slot("a0", 512, 768, 4, 0), li.Slot("b0", 768, 512, 4, 1),
                               li.Slot("a1", 512, 768, 4, 2), li.Slot("b1", 768, 512, 4, 3)), 64, 24, 4, 2, 250, "bf16")
    b = li.make_batch(cfg)
    T = b.n_rows
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots], [4] * 4, cfg.rank,
                      cfg.n_adapters, cfg.scale(), T, 0, expert_parallel=True, pp_stages=2, slot_layer=[0, 0, 1, 1])
    s = B.lora_server_create(c)
    try:
        B.lora_server_fill_synthetic(s, cfg.seed)
        my_layer = rank // 2
        for layer in (0, 1):
            sl = [2 * layer, 2 * layer + 1]
            if layer != my_layer:
                with pytest.raises(B.LoraError):
                    _run_multi_unchecked(B, s, cfg, b, sl)
                continue
            own = orc.owner_of(b.adapter_ids, 4, 0, None, b.expert_ids, True, 2, layer)
            y0 = [U.y0_dev(B, cfg, i, T) for i in sl]
            ys = _run_multi_unchecked(B, s, cfg, b, sl)
            assert B.lora_server_check(s) == B.LORA_ERR_ID_OUT_OF_RANGE   # the other rank's rows
            rows = np.flatnonzero(own == rank)
            other = torch.from_numpy(np.flatnonzero(own != rank)).to(U.DEV)
            assert rows.size > 0
            for j, i in enumerate(sl):
                U.assert_parity(ys[j][torch.from_numpy(rows).to(U.DEV)], oracle.apply_slot(cfg, i, b, rows=rows),
                                f"hybrid rank {rank} slot {i}")
                assert torch.equal(ys[j][other], y0[j][other])
    finally:
        B.lora_server_destroy(s)
