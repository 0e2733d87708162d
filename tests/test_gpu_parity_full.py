"""GPU parity at full size, every row, and the harder input distributions.

- every row of every slot of BASELINE.json configs 2-5 against the oracle, in
  the launch configuration bench.py times (one plan, one multi-slot apply; all
  128 Llama slots in one launch), with a random base output y0 AND with y0 = 0
  so that the north-star bound max|err| <= 1e-2*max|y| + 1e-3 binds on the
  delta itself (SURVEY 8c reading #12);
- full-mantissa, wide-exponent bf16 inputs (x ~ N(0,1), A ~ N(0,1/h_in),
  B ~ N(0,1/r), y0 ~ N(0,1)) loaded through lora_server_create's
  host weights, on both tcgen05 shrink routes (K-split for decode-sized
  batches, whole-K for T >= 4096) and the CUDA-core route;
- exact-integer probes (bit-exact whatever the summation order) on the
  whole-K tcgen05 route at T >= 4096, with an fp32 and a bf16 output, and
  with 128 / 130 slots in one call (task tables, launch batching);
- the sharded server's handling of a bad expert id on a routed row, both
  transports;
- lora_server_load: partial adapter ranges from host and device memory, and
  a sharded (fake-world) store skipping adapters the rank does not own;
- cross-slot x / y aliasing rejected with nothing enqueued.
"""
import dataclasses

import numpy as np
import pytest
import torch

import lora_inputs as li
from oracle import oracle as orc

from tests import gpu_util as U

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    return U.binding()


def _run(B, s, cfg, batch, slot_ids, y0):
    T = batch.n_rows
    ad, ex = U.ids_dev(batch)
    E = cfg.slots[slot_ids[0]].n_experts
    xs = {}
    for i in slot_ids:
        if cfg.slots[i].xbuf not in xs:
            xs[cfg.slots[i].xbuf] = U.x_dev(B, cfg, i, T)
    ys = [U.y0_dev(B, cfg, i, T, y0) for i in slot_ids]
    dt = B.LORA_FP32 if cfg.y_dtype == "fp32" else B.LORA_BF16
    p = B.lora_plan_create(s, T)
    try:
        B.lora_plan_build(s, p, ad, ex if E > 1 else None, T, E)
        B.lora_apply_plan_multi(s, p, list(slot_ids), [xs[cfg.slots[i].xbuf] for i in slot_ids], ys, dt)
        torch.cuda.synchronize()
        assert B.lora_server_check(s) == B.LORA_OK
        stats = B.lora_plan_stats(s, p)
    finally:
        B.lora_plan_destroy(p)
    return ys, stats


# ---------------------------------------------------------------------------
# every row, configs 2-5
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["llama_decode", "mixtral_decode", "mixtral_prefill", "mixtral_sharded",
                                  "mixtral_decode_uniform", "llama_decode_uniform", "mixtral_prefill_16x512"])
def test_full_config_every_row(B, name):
    cfg = li.CONFIGS[name] if name in li.CONFIGS else li.VARIANTS[name]
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    slots = list(range(len(cfg.slots)))
    try:
        for y0 in ("random", "zero"):
            ys, stats = _run(B, s, cfg, b, slots, y0)
            if name in li.CONFIGS and cfg.rank == 64:
                assert stats[3] > 0, stats                    # the tcgen05 route ran
                assert stats[2] > 0 or name == "mixtral_prefill", stats   # (prefill: every segment is large)
            for i in slots:
                ref = orc.apply_slot_all_rows(cfg, i, b, y0=y0)
                U.assert_parity(ys[i], ref, f"{name} slot {i} y0={y0}")
                if y0 == "random":  # rows without a LoRA: bit-identical (none in these configs' ids)
                    none = np.flatnonzero(b.adapter_ids < 0)
                    assert none.size == 0 or torch.equal(
                        ys[i][torch.from_numpy(none).to(U.DEV)],
                        U.y0_dev(B, cfg, i, b.n_rows)[torch.from_numpy(none).to(U.DEV)])
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("rank", [8, 32, 128])
def test_prefill_shapes_other_ranks_every_row(B, rank):
    """Config 4's shapes (Mixtral gate/up/down, 8192 tokens, 16384 rows) at
    r = 32 and r = 128: the tcgen05 chain at those ranks (SWIZZLE_64B operands;
    r = 128: two K blocks, Bt re-tiled in the expand's producer), whole-K
    items, the paired gate/up shrink; every row against the oracle."""
    cfg = dataclasses.replace(li.CONFIGS["mixtral_prefill"], name=f"mixtral_prefill_r{rank}", rank=rank)
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    slots = list(range(len(cfg.slots)))
    try:
        ys, stats = _run(B, s, cfg, b, slots, "random")
        assert stats[3] > 0, stats  # the tcgen05 route ran
        for i in slots:
            U.assert_parity(ys[i], orc.apply_slot_all_rows(cfg, i, b, y0="random"), f"prefill r={rank} slot {i}")
    finally:
        B.lora_server_destroy(s)


def test_config5_push_loopback_every_row(B, monkeypatch):
    """Config 5 through the sharded server's push path at full size
    (loopback: every row through bucket / announce / recv-prep, the owner's
    remote-x shrink and the push-add expand), every row against the oracle."""
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
        for y0 in ("random", "zero"):
            for i in range(3):
                ys[i].copy_(U.y0_dev(B, cfg, i, T, y0))
            B.lora_apply_sharded(sh, [0, 1, 2], [xs[sl.xbuf] for sl in cfg.slots], ad, ex, ys, B.LORA_BF16, T)
            torch.cuda.synchronize()
            assert B.lora_server_check(sh) == B.LORA_OK
            for i in range(3):
                U.assert_parity(ys[i], orc.apply_slot_all_rows(cfg, i, b, y0=y0), f"p2p loopback slot {i} y0={y0}")
    finally:
        B.lora_server_destroy(sh)


# ---------------------------------------------------------------------------
# full-mantissa N(0,1)-style inputs through host weights
# ---------------------------------------------------------------------------
def _normal_problem(seed, slots, rank, n_ad, E, n_tokens, top_k, zipf=1.2):
    rng = np.random.default_rng(seed)
    A = [li.normal_bf16_bits(rng, (n_ad, E, hi, rank), 1.0 / np.sqrt(hi)) for hi, ho in slots]
    Bw = [li.normal_bf16_bits(rng, (n_ad, E, rank, ho), 1.0 / np.sqrt(rank)) for hi, ho in slots]
    # Zipf over adapters [0, n_ad-1); the last adapter gets a dozen tokens, so
    # small segments (CUDA-core route) exist even in large batches
    tok = rng.choice(n_ad - 1, size=n_tokens, p=li.zipf_probs(n_ad - 1, zipf)).astype(np.int32)
    tok[rng.choice(n_tokens, min(12, n_tokens), replace=False)] = n_ad - 1
    tok[rng.random(n_tokens) < 0.03] = -1
    ad = np.repeat(tok, top_k).astype(np.int32)
    ex = (np.argsort(rng.random((n_tokens, E)), axis=1)[:, :top_k].reshape(-1).astype(np.int32)
          if E > 1 else np.zeros(n_tokens * top_k, np.int32))
    T = n_tokens * top_k
    x = {hi: li.normal_bf16_bits(rng, (T, hi)) for hi, _ in slots}
    y0 = [li.normal_bf16_bits(rng, (T, ho)) for _, ho in slots]
    scale = np.array([(0.5, 1.0, 2.0)[a % 3] for a in range(n_ad)], np.float32)
    return A, Bw, ad, ex, x, y0, scale


@pytest.mark.parametrize("case", ["mixtral_wholek", "mixtral_ksplit", "llama_r16"])
def test_full_mantissa_inputs(B, case):
    if case == "llama_r16":
        slots, rank, n_ad, E, n_tok, k = [(4096, 4096), (4096, 1024)], 16, 32, 1, 256, 1
    else:
        slots, rank, n_ad, E, k = [(4096, 14336), (14336, 4096)], 64, 12, 8, 2
        n_tok = 4096 if case == "mixtral_wholek" else 400
    A, Bw, ad, ex, x, y0s, scale = _normal_problem(7, slots, rank, n_ad, E, n_tok, k)
    T = ad.size
    c = B.make_config([hi for hi, _ in slots], [ho for _, ho in slots], [E] * len(slots), rank, n_ad, scale, T, 0)
    s = B.lora_server_create(c, A, Bw, weights_on_device=False)
    try:
        p = B.lora_plan_create(s, T)
        B.lora_plan_build(s, p, torch.from_numpy(ad).to(U.DEV), torch.from_numpy(ex).to(U.DEV) if E > 1 else None,
                          T, E)
        stats = B.lora_plan_stats(s, p)
        if rank == 64:
            assert stats[2] > 0 and stats[3] > 0, stats
        xd = [torch.from_numpy(x[hi].view(np.int16)).to(U.DEV) for hi, _ in slots]
        uor, units, sor = orc.unit_tables(ad, ex, E, n_ad, scale)
        for zero in (False, True):
            ys = [torch.zeros((T, ho), dtype=torch.int16, device=U.DEV) if zero
                  else torch.from_numpy(y0s[i].view(np.int16)).to(U.DEV) for i, (_, ho) in enumerate(slots)]
            B.lora_apply_plan_multi(s, p, list(range(len(slots))), xd, ys, B.LORA_BF16)
            torch.cuda.synchronize()
            assert B.lora_server_check(s) == B.LORA_OK
            for i, (hi, ho) in enumerate(slots):
                a_u, e_u = units // E, units % E
                Au = A[i][a_u, e_u] if units.size else np.zeros((0, hi, rank), np.uint16)
                Bu = Bw[i][a_u, e_u] if units.size else np.zeros((0, rank, ho), np.uint16)
                yref = np.zeros((T, ho), np.uint16) if zero else y0s[i].copy()
                orc.lora_apply_rows(x[hi], uor, sor, Au, Bu, yref)
                U.assert_parity(ys[i], yref, f"{case} slot {i} zero={zero}")
        B.lora_plan_destroy(p)
    finally:
        B.lora_server_destroy(s)


# ---------------------------------------------------------------------------
# exact-integer probes: whole-K tcgen05 route (T >= 4096), bf16 output, many slots
# ---------------------------------------------------------------------------
def _int_server(B, shapes, rank, n_ad, E, T, rng, b_sparse=False):
    scale = np.array([(0.5, 1.0, 2.0)[i % 3] for i in range(n_ad)], np.float32)
    bits = lambda v: li.f32_to_bf16_bits_exact(np.asarray(v, np.float32))
    Ai = [rng.integers(-1, 2, (n_ad * E, hi, rank)) for hi, _ in shapes]
    if b_sparse:  # one nonzero (+-1) per output column: |delta| <= 2 |v|_max
        Bi = []
        for _, ho in shapes:
            m = np.zeros((n_ad * E, rank, ho), np.int64)
            kk = rng.integers(0, rank, (n_ad * E, ho))
            m[np.arange(n_ad * E)[:, None], kk, np.arange(ho)[None, :]] = rng.choice([-1, 1], (n_ad * E, ho))
            Bi.append(m)
    else:
        Bi = [rng.integers(-1, 2, (n_ad * E, rank, ho)) for _, ho in shapes]
    c = B.make_config([hi for hi, _ in shapes], [ho for _, ho in shapes], [E] * len(shapes), rank, n_ad, scale, T, 0)
    s = B.lora_server_create(c, [bits(a) for a in Ai], [bits(b) for b in Bi], weights_on_device=False)
    return s, Ai, Bi, scale, bits


def _sparse_x(rng, T, h_in, nnz):
    """Integer rows with nnz nonzeros in {-2,-1,1,2} spread over the whole row,
    so |v| <= 2*nnz stays exact in bf16 (v is a bf16 MMA operand on tcgen05)."""
    x = np.zeros((T, h_in), np.int64)
    for i in range(T):
        pos = rng.choice(h_in, nnz, replace=False)
        x[i, pos] = rng.choice([-2, -1, 1, 2], nnz)
    return x


def _int_expect(xi, y0, a, e, E, Ai, Bi, scale):
    exp = y0.astype(np.float64).copy()
    for i in range(len(a)):
        if a[i] >= 0:
            u = a[i] * E + e[i]
            exp[i] += float(scale[a[i]]) * ((xi[i] @ Ai[u]) @ Bi[u])
    return exp


@pytest.mark.parametrize("y_dtype", ["fp32", "bf16"])
def test_exact_integer_probes_wholek_large_batch(B, y_dtype):
    rng = np.random.default_rng(41 if y_dtype == "fp32" else 42)
    E, n_ad, T = 2, 8, 4400
    shapes = [(2048, 256), (1024, 384)]
    s, Ai, Bi, scale, bits = _int_server(B, shapes, 64, n_ad, E, T, rng, b_sparse=(y_dtype == "bf16"))
    try:
        a = rng.choice(np.arange(-1, n_ad - 1), T, p=[0.02] + [0.98 / (n_ad - 1)] * (n_ad - 1)).astype(np.int32)
        a[:300] = 3                      # one large segment per expert
        a[300:310] = n_ad - 1            # ~5 rows per expert: CUDA-core groups
        e = rng.integers(0, E, T).astype(np.int32)
        p = B.lora_plan_create(s, T)
        B.lora_plan_build(s, p, torch.from_numpy(a).to(U.DEV), torch.from_numpy(e).to(U.DEV), T, E)
        nv, ns, ng, nt = B.lora_plan_stats(s, p)
        assert nt > 0 and ng > 0
        nnz = 96 if y_dtype == "fp32" else 16
        xs, ys, exps = [], [], []
        for hi, ho in shapes:
            xi = _sparse_x(rng, T, hi, nnz)
            xs.append(torch.from_numpy(bits(xi).view(np.int16)).to(U.DEV))
            lim = 50 if y_dtype == "fp32" else 32
            yi = rng.integers(-lim, lim + 1, (T, ho)).astype(np.float32)
            ys.append(torch.from_numpy(yi.copy()).to(U.DEV) if y_dtype == "fp32"
                      else torch.from_numpy(bits(yi).view(np.int16)).to(U.DEV))
            exps.append((xi, yi))
        B.lora_apply_plan_multi(s, p, [0, 1], xs, ys, B.LORA_FP32 if y_dtype == "fp32" else B.LORA_BF16)
        torch.cuda.synchronize()
        B.lora_plan_destroy(p)
        for i in range(2):
            xi, yi = exps[i]
            exp = _int_expect(xi, yi, a, e, E, Ai[i], Bi[i], scale).astype(np.float32)
            got = ys[i].cpu().numpy() if y_dtype == "fp32" else li.bf16_bits_to_f32(ys[i].cpu().numpy().view(np.uint16))
            if y_dtype == "bf16":
                assert np.abs(exp).max() < 128                    # exact in bf16 by construction
            np.testing.assert_array_equal(got, exp)
    finally:
        B.lora_server_destroy(s)


@pytest.mark.parametrize("rank,n_slots", [(16, 128), (64, 128), (16, 130)])
def test_exact_integer_probes_many_slots(B, rank, n_slots):
    """128 slots in one call (the Llama decode step's launch), and 130 (two
    launch batches of <= 128 tasks), bit-exact."""
    rng = np.random.default_rng(rank + n_slots)
    E, n_ad, T = 1, 10, 300
    shapes = [(128, (128, 256, 128, 384)[i % 4]) for i in range(n_slots)]
    s, Ai, Bi, scale, bits = _int_server(B, shapes, rank, n_ad, E, T, rng)
    try:
        a = rng.integers(-1, n_ad, T).astype(np.int32)
        a[:100] = 2
        e = np.zeros(T, np.int32)
        xi = rng.integers(-2, 3, (T, 128))
        x = torch.from_numpy(bits(xi).view(np.int16)).to(U.DEV)
        y0 = [rng.integers(-50, 51, (T, ho)).astype(np.float32) for _, ho in shapes]
        ys = [torch.from_numpy(v.copy()).to(U.DEV) for v in y0]
        p = B.lora_plan_create(s, T)
        B.lora_plan_build(s, p, torch.from_numpy(a).to(U.DEV), None, T, 1)
        B.lora_apply_plan_multi(s, p, list(range(n_slots)), [x] * n_slots, ys, B.LORA_FP32)
        torch.cuda.synchronize()
        B.lora_plan_destroy(p)
        for i in range(n_slots):
            exp = _int_expect(xi, y0[i], a, e, E, Ai[i], Bi[i], scale).astype(np.float32)
            np.testing.assert_array_equal(ys[i].cpu().numpy(), exp, err_msg=f"slot {i}")
    finally:
        B.lora_server_destroy(s)


# ---------------------------------------------------------------------------
# boundary: sharded bad expert id, lora_server_load, cross-slot aliasing
# ---------------------------------------------------------------------------
def _mid_cfg(rank=64, T=600, y_dtype="bf16"):
    return li.Config("mid", 8, (li.Slot("a", 512, 768, 4, 0), li.Slot("b", 768, 512, 4, 1)), rank, 24, 4, 2,
                     T // 2, y_dtype)


@pytest.mark.parametrize("transport", ["push", "nccl"])
def test_sharded_bad_expert_id_on_routed_row(B, monkeypatch, transport):
    """A routed row (loopback: every row is routed) with a valid adapter and an
    out-of-range expert id is flagged and dropped: its y row is unchanged, the
    other rows match the unsharded server, lora_server_check reports it."""
    monkeypatch.setenv("LORA_SHARD_LOOPBACK", "1")
    cfg = _mid_cfg(y_dtype="fp32")
    b = li.make_batch(cfg)
    T = b.n_rows
    ex_bad = b.expert_ids.copy()
    bad_rows = [5, 77]
    ex_bad[5] = 4      # E = 4: out of range
    ex_bad[77] = -3
    b.adapter_ids[bad_rows] = [1, 2]
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                      [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(), T, 0)
    sh = B.lora_server_create_sharded(c, 0, 1, B.lora_nccl_unique_id())
    s = U.make_server(B, cfg)
    try:
        B.lora_server_fill_synthetic(sh, cfg.seed)
        good = li.Batch(np.where(np.isin(np.arange(T), bad_rows), -1, b.adapter_ids).astype(np.int32),
                        b.expert_ids, b.n_tokens, b.top_k)
        y_ref, _ = _run(B, s, cfg, good, [0, 1], "random")
        ad = torch.from_numpy(b.adapter_ids).to(U.DEV)
        ex = torch.from_numpy(ex_bad).to(U.DEV)
        xs = [U.x_dev(B, cfg, i, T) for i in range(2)]
        ys = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        if transport == "push":
            U.register(B, sh, xs + ys)
        for rep in range(2):   # the second call must not see a stale delta either
            for i in range(2):
                ys[i].copy_(U.y0_dev(B, cfg, i, T))
            B.lora_apply_sharded(sh, [0, 1], xs, ad, ex, ys, B.LORA_FP32, T)
            torch.cuda.synchronize()
            assert B.lora_server_check(sh) == B.LORA_ERR_ID_OUT_OF_RANGE
            for i in range(2):
                y0 = U.y0_dev(B, cfg, i, T)
                for r in bad_rows:
                    assert torch.equal(ys[i][r].view(torch.int32), y0[r].view(torch.int32))
                assert torch.equal(ys[i].view(torch.int32), y_ref[i].view(torch.int32))
    finally:
        B.lora_server_destroy(sh)
        B.lora_server_destroy(s)


def test_server_load_partial_ranges_host_and_device(B):
    """lora_server_load of adapter ranges [0,5) from host, [5,17) from device,
    [17,24) from host (A only, then B only) == lora_server_create with all
    weights (bit-identical y), for both kernel routes."""
    cfg = _mid_cfg()
    rng = np.random.default_rng(5)
    E, n_ad, r = 4, cfg.n_adapters, cfg.rank
    A = [li.normal_bf16_bits(rng, (n_ad, E, sl.h_in, r), 0.05) for sl in cfg.slots]
    Bw = [li.normal_bf16_bits(rng, (n_ad, E, r, sl.h_out), 0.1) for sl in cfg.slots]
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots], [E, E], r, n_ad, cfg.scale(),
                      cfg.n_rows, 0)
    full = B.lora_server_create(c, A, Bw, weights_on_device=False)
    ld = B.lora_server_create(c)
    try:
        for i in range(2):
            B.lora_server_load(ld, i, 0, 5, A[i][:5], Bw[i][:5], on_device=False)
            Ad = torch.from_numpy(A[i][5:17].view(np.int16)).to(U.DEV)
            Bd = torch.from_numpy(Bw[i][5:17].view(np.int16)).to(U.DEV)
            B.lora_server_load(ld, i, 5, 12, Ad, Bd, on_device=True)
            B.lora_server_load(ld, i, 17, 7, np.ascontiguousarray(A[i][17:]), None, on_device=False)
            B.lora_server_load(ld, i, 17, 7, None, np.ascontiguousarray(Bw[i][17:]), on_device=False)
        with pytest.raises(B.LoraError):
            B.lora_server_load(ld, 0, 20, 5, A[0][:5], Bw[0][:5], on_device=False)   # past n_adapters
        b = li.make_batch(cfg)
        for sm in (None, -1):
            if sm is not None:
                B.lora_server_set_small_seg_max(full, sm)
                B.lora_server_set_small_seg_max(ld, sm)
            y1, _ = _run(B, full, cfg, b, [0, 1], "random")
            y2, _ = _run(B, ld, cfg, b, [0, 1], "random")
            for i in range(2):
                assert torch.equal(y1[i], y2[i])
    finally:
        B.lora_server_destroy(full)
        B.lora_server_destroy(ld)


@pytest.mark.parametrize("ep,n_hot", [(0, 0), (0, 3), (1, 0)])
def test_server_load_sharded_skips_unowned(B, monkeypatch, ep, n_hot):
    """lora_server_load on rank 1 of a 2-rank (fake-world) server stores only
    the units that rank owns; its owned rows equal the full server's."""
    monkeypatch.setenv("LORA_FAKE_WORLD", f"2,1,{ep},{n_hot}")
    cfg = _mid_cfg(rank=16, y_dtype="fp32")
    rng = np.random.default_rng(9)
    E, n_ad, r = 4, cfg.n_adapters, cfg.rank
    A = [li.normal_bf16_bits(rng, (n_ad, E, sl.h_in, r), 0.05) for sl in cfg.slots]
    Bw = [li.normal_bf16_bits(rng, (n_ad, E, r, sl.h_out), 0.1) for sl in cfg.slots]
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots], [E, E], r, n_ad, cfg.scale(),
                      cfg.n_rows, 0)
    ld = B.lora_server_create(c)
    monkeypatch.delenv("LORA_FAKE_WORLD")
    full = B.lora_server_create(c, A, Bw, weights_on_device=False)
    try:
        for i in range(2):
            B.lora_server_load(ld, i, 0, 10, A[i][:10], Bw[i][:10], on_device=False)
            B.lora_server_load(ld, i, 10, 14, A[i][10:], Bw[i][10:], on_device=False)
        b = li.make_batch(cfg)
        own = orc.owner_of(b.adapter_ids, 2, n_hot, np.full(b.n_rows, 1), b.expert_ids, bool(ep))
        y_full, _ = _run(B, full, cfg, b, [0, 1], "random")
        T = b.n_rows
        ad, ex = U.ids_dev(b)
        xs = [U.x_dev(B, cfg, i, T) for i in range(2)]
        ys = [U.y0_dev(B, cfg, i, T) for i in range(2)]
        p = B.lora_plan_create(ld, T)
        B.lora_plan_build(ld, p, ad, ex, T, E)
        B.lora_apply_plan_multi(ld, p, [0, 1], xs, ys, B.LORA_FP32)
        torch.cuda.synchronize()
        B.lora_plan_destroy(p)
        B.lora_server_check(ld)
        mine = torch.from_numpy(np.flatnonzero(own == 1)).to(U.DEV)
        assert mine.numel() > 0
        for i in range(2):
            assert torch.equal(ys[i][mine], y_full[i][mine])
    finally:
        B.lora_server_destroy(ld)
        B.lora_server_destroy(full)


def test_cross_slot_aliasing_rejected(B):
    cfg = _mid_cfg(T=64)
    b = li.make_batch(cfg)
    s = U.make_server(B, cfg)
    try:
        T = b.n_rows
        ad, ex = U.ids_dev(b)
        p = B.lora_plan_create(s, T)
        B.lora_plan_build(s, p, ad, ex, T, 4)
        x0 = U.x_dev(B, cfg, 0, T)
        x1 = U.x_dev(B, cfg, 1, T)
        big = torch.zeros(T * 768 * 3, dtype=torch.int16, device=U.DEV)
        y0 = big[:T * 768]
        y1 = big[T * 768:T * 768 + T * 512]
        before = big.clone()
        # slot 1's y is slot 0's x buffer
        with pytest.raises(B.LoraError):
            B.lora_apply_plan_multi(s, p, [0, 1], [x0, x1], [y0, x0.view(-1)[:T * 512]], B.LORA_BF16)
        # two y ranges overlapping
        with pytest.raises(B.LoraError):
            B.lora_apply_plan_multi(s, p, [0, 1], [x0, x1], [y0, big[T * 700:T * 700 + T * 512]], B.LORA_BF16)
        # slot 0's y overlapping slot 1's x
        y1_sep = torch.zeros(T * 512, dtype=torch.int16, device=U.DEV)
        with pytest.raises(B.LoraError):
            B.lora_apply_plan_multi(s, p, [0, 1], [x0, big[T * 100:T * 100 + T * 768]], [y0, y1_sep], B.LORA_BF16)
        torch.cuda.synchronize()
        assert torch.equal(big, before)        # nothing was enqueued
        # disjoint buffers and a shared x are accepted
        B.lora_apply_plan_multi(s, p, [0, 1], [x0, x1], [y0, y1], B.LORA_BF16)
        torch.cuda.synchronize()
        B.lora_plan_destroy(p)
    finally:
        B.lora_server_destroy(s)


def test_tc_min_rows_heuristic(B, monkeypatch):
    """Default LORA_TC_MIN_ROWS (256): with fewer rows than that in large
    segments every segment takes the CUDA-core route (no tcgen05 tiles); with
    more, the large segments go to tcgen05.  Results within the oracle's
    tolerance either way."""
    monkeypatch.delenv("LORA_TC_MIN_ROWS", raising=False)
    cfg = _mid_cfg(T=400)
    s = U.make_server(B, cfg)
    try:
        for n_big, want_tiles in ((100, False), (300, True)):
            T = 400
            a = np.arange(T, dtype=np.int32) % cfg.n_adapters   # small segments
            a[:n_big] = 5
            e = (np.arange(T, dtype=np.int32) // cfg.n_adapters) % 4   # 96 keys of <= 5 rows
            e[:n_big] = 1
            b = li.Batch(a, e, T, 1)
            c2 = dataclasses.replace(cfg, top_k=1, n_tokens=T)
            ys, stats = _run(B, s, c2, b, [0, 1], "random")
            assert (stats[3] > 0) == want_tiles, (n_big, stats)
            for i in range(2):
                U.assert_parity(ys[i], orc.apply_slot(c2, i, b), f"min-rows {n_big} slot {i}")
    finally:
        B.lora_server_destroy(s)


def test_host_entry_row_chunks(B, monkeypatch):
    """lora_apply_multi_host with several row chunks (a 4100-row batch: two
    chunks, one plan each, pieces of (row chunk, slot group) pipelined over
    the copy engines) against the oracle, rows without a LoRA bit-identical."""
    cfg = dataclasses.replace(_mid_cfg(T=4100), no_lora_frac=0.05)
    b = li.make_batch(cfg)
    T = b.n_rows
    s = U.make_server(B, cfg)
    try:
        xh = [U.x_dev(B, cfg, i, T).cpu().pin_memory() for i in range(2)]
        yh = [U.y0_dev(B, cfg, i, T).cpu().pin_memory() for i in range(2)]
        y0 = [y.clone() for y in yh]
        B.lora_apply_multi_host(s, [0, 1], xh, b.adapter_ids, b.expert_ids, yh, B.LORA_BF16, T)
        torch.cuda.synchronize()
        assert B.lora_server_check(s) == B.LORA_OK
        none = torch.from_numpy(np.flatnonzero(b.adapter_ids < 0))
        assert none.numel() > 0
        for i in range(2):
            U.assert_parity(yh[i], orc.apply_slot(cfg, i, b), f"host row chunks slot {i}")
            assert torch.equal(yh[i][none], y0[i][none])
    finally:
        B.lora_server_destroy(s)


# ---------------------------------------------------------------------------
# the delta API (the server returns s_a (x A) B; the client adds)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype,T", [("bf16", 600), ("fp32", 600), ("bf16", 4200), ("fp32", 4200)])
def test_delta_api_equals_apply_on_zero_y(B, dtype, T):
    """lora_apply_plan_multi_delta equals lora_apply_plan_multi on a zero y
    bit for bit (both kernel chains, K-split and whole-K tcgen05 items), rows
    without a LoRA get a zero delta even in a dirty output buffer, and the
    deltas match the oracle's y0 = 0 result."""
    cfg = dataclasses.replace(_mid_cfg(T=T), no_lora_frac=0.05, y_dtype=dtype)
    b = li.make_batch(cfg)
    Tr = b.n_rows
    s = U.make_server(B, cfg)
    dt = B.LORA_FP32 if dtype == "fp32" else B.LORA_BF16
    tdt = torch.float32 if dtype == "fp32" else torch.int16
    try:
        ad, ex = U.ids_dev(b)
        xs = [U.x_dev(B, cfg, i, Tr) for i in range(2)]
        p = B.lora_plan_create(s, Tr)
        B.lora_plan_build(s, p, ad, ex, Tr, 4)
        ys = [torch.zeros((Tr, sl.h_out), dtype=tdt, device=U.DEV) for sl in cfg.slots]
        B.lora_apply_plan_multi(s, p, [0, 1], xs, ys, dt)
        ds = [torch.full((Tr, sl.h_out), 7, dtype=tdt, device=U.DEV) for sl in cfg.slots]  # dirty
        B.lora_apply_plan_multi_delta(s, p, [0, 1], xs, ds, dt)
        torch.cuda.synchronize()
        assert B.lora_server_check(s) == B.LORA_OK
        B.lora_plan_destroy(p)
        none = torch.from_numpy(np.flatnonzero(b.adapter_ids < 0)).to(U.DEV)
        assert none.numel() > 0
        for i in range(2):
            assert torch.equal(ds[i], ys[i]), f"slot {i}"
            assert not ds[i][none].any()
            U.assert_parity(ds[i], orc.apply_slot(cfg, i, b, y0="zero"), f"delta {dtype} slot {i}")
    finally:
        B.lora_server_destroy(s)


def test_host_delta_equals_host_apply_on_zero_y(B):
    """lora_apply_multi_host_delta (x and ids up, deltas down, row-chunked
    pipeline) equals lora_apply_multi_host on a zero y bit for bit."""
    cfg = dataclasses.replace(_mid_cfg(T=4100), no_lora_frac=0.05)
    b = li.make_batch(cfg)
    T = b.n_rows
    s = U.make_server(B, cfg)
    try:
        xh = [U.x_dev(B, cfg, i, T).cpu().pin_memory() for i in range(2)]
        yh = [torch.zeros((T, sl.h_out), dtype=torch.int16).pin_memory() for sl in cfg.slots]
        dh = [torch.full((T, sl.h_out), 3, dtype=torch.int16).pin_memory() for sl in cfg.slots]
        B.lora_apply_multi_host(s, [0, 1], xh, b.adapter_ids, b.expert_ids, yh, B.LORA_BF16, T)
        B.lora_apply_multi_host_delta(s, [0, 1], xh, b.adapter_ids, b.expert_ids, dh, B.LORA_BF16, T)
        torch.cuda.synchronize()
        assert B.lora_server_check(s) == B.LORA_OK
        for i in range(2):
            assert torch.equal(dh[i], yh[i]), f"slot {i}"
    finally:
        B.lora_server_destroy(s)


def test_server_reuse_across_batch_sizes(B):
    """One server and one plan reused across batches of very different sizes
    (1 to 20000 rows: one-CTA and multi-CTA segmenter, K-split and whole-K
    tcgen05 items, CUDA-core only, no-LoRA rows) in one stream: the
    self-resetting device state (work counters, histograms, arrival counters)
    carries no stale value from one build / apply to the next."""
    base = _mid_cfg(T=20000)
    s = U.make_server(B, base)  # max_rows = 20000
    p = B.lora_plan_create(s, base.n_rows)
    try:
        for k, n_tok in enumerate((10000, 1, 300, 7, 2100, 10000, 64, 4100)):
            cfg = dataclasses.replace(base, n_tokens=n_tok, no_lora_frac=0.05 * (k % 2))
            b = li.make_batch(cfg, seed=50 + k)
            T = b.n_rows
            ad, ex = U.ids_dev(b)
            xs = [U.x_dev(B, cfg, i, T) for i in range(2)]
            ys = [U.y0_dev(B, cfg, i, T) for i in range(2)]
            B.lora_plan_build(s, p, ad, ex, T, 4)
            B.lora_apply_plan_multi(s, p, [0, 1], xs, ys, B.LORA_BF16)
            torch.cuda.synchronize()
            assert B.lora_server_check(s) == B.LORA_OK
            for i in range(2):
                U.assert_parity(ys[i], orc.apply_slot(cfg, i, b), f"reuse step {k} ({T} rows) slot {i}")
    finally:
        B.lora_plan_destroy(p)
        B.lora_server_destroy(s)
