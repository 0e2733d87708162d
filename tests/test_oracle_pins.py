"""Pins of the CPU oracle against things other than itself (CPU only).

Each test fixes the oracle to an independent source of truth: a hand-worked
golden example (tests/golden, cited), the dense merged-weight form
W' = W + s*A*B of P:165 evaluated by numpy in float64, its PEFT-transposed
form, exact integer arithmetic (numpy int64 matmul), rank-1 outer products,
library bf16 rounding (torch), invariants (a = -1, permutation, linearity in
s, thread count) and, for the segmenter, a pure-Python sorted()/groupby brute
force.  See DESIGN.md "Oracle and pins".
"""
import itertools
import json
import os

import numpy as np
import pytest

import lora_inputs as li
import oracle
from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _bits(f):
    return li.f32_to_bf16_bits_exact(np.asarray(f, np.float32))


def _rand_bf16(rng, shape, lo=-2.0, hi=2.0, step=2 ** -5):
    """bf16-exact random values (few significant bits)."""
    q = rng.integers(int(lo / step), int(hi / step), size=shape)
    return (q * step).astype(np.float32)


# ---------------------------------------------------------------------------
# golden, hand-worked
# ---------------------------------------------------------------------------
def test_golden_hand_example():
    g = json.load(open(os.path.join(GOLDEN, "delta_hand.json")))
    E = g["n_experts"]
    a = np.array(g["adapter_ids"], np.int32)
    e = np.array(g["expert_ids"], np.int32)
    uor, units, sor = orc.unit_tables(a, e, E, g["n_adapters"], np.array(g["scale"], np.float32))
    A = np.stack([_bits(g["units"][str(int(u))]["A"]) for u in units])
    B = np.stack([_bits(g["units"][str(int(u))]["B"]) for u in units])
    y = np.array(g["y0"], np.float32)
    orc.lora_apply_rows(_bits(g["x"]), uor, sor, A, B, y)
    np.testing.assert_array_equal(y, np.array(g["y_expected"], np.float32))
    # same, bf16 output (all values exact in bf16)
    yb = _bits(g["y0"])
    orc.lora_apply_rows(_bits(g["x"]), uor, sor, A, B, yb)
    np.testing.assert_array_equal(li.bf16_bits_to_f32(yb), np.array(g["y_expected"], np.float32))


def test_bf16_rounding_ties_to_even_and_library():
    # hand: ulp(1.0) in bf16 is 2^-7; 1 + 2^-8 is a tie -> even (1.0); 1 + 3*2^-8 -> 1 + 2^-6
    assert orc.round_bf16(1.0 + 2 ** -8) == 0x3F80
    assert orc.round_bf16(1.0 + 3 * 2 ** -8) == 0x3F82
    assert orc.round_bf16(-(1.0 + 3 * 2 ** -8)) == 0xBF82
    assert orc.round_bf16(0.0) == 0 and orc.round_bf16(-0.0) == 0x8000
    assert orc.round_bf16(1e39) == 0x7F80
    # library pin: torch's float32 -> bfloat16 cast is RNE; compare on float32 values
    import torch
    rng = np.random.default_rng(0)
    f = (rng.standard_normal(20000) * 10.0 ** rng.integers(-30, 30, 20000)).astype(np.float32)
    ref = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().astype(np.uint16)
    got = np.array([orc.round_bf16(float(v)) for v in f], np.uint16)
    np.testing.assert_array_equal(got, ref)


# ---------------------------------------------------------------------------
# dense brute force (merged weights, float64 numpy)
# ---------------------------------------------------------------------------
def _random_problem(rng, T=40, h_in=16, h_out=12, r=4, n_ad=5, E=3, no_lora=0.2):
    a = rng.integers(0, n_ad, T).astype(np.int32)
    a[rng.random(T) < no_lora] = -1
    e = rng.integers(0, E, T).astype(np.int32)
    A = _rand_bf16(rng, (n_ad * E, h_in, r), -0.5, 0.5, 2 ** -7)
    B = _rand_bf16(rng, (n_ad * E, r, h_out), -0.5, 0.5, 2 ** -7)
    x = _rand_bf16(rng, (T, h_in))
    s = np.array([0.5, 1.0, 2.0, 0.25, 1.5][:n_ad], np.float32)
    y0 = _rand_bf16(rng, (T, h_out))
    return a, e, A, B, x, s, y0


def _oracle_full(a, e, A, B, x, s, y0, E, n_ad, y_bits=False, threads=0):
    uor, units, sor = orc.unit_tables(a, e, E, n_ad, s)
    Au = np.stack([_bits(A[u]) for u in units]) if units.size else np.zeros((0,) + A.shape[1:], np.uint16)
    Bu = np.stack([_bits(B[u]) for u in units]) if units.size else np.zeros((0,) + B.shape[1:], np.uint16)
    y = _bits(y0) if y_bits else y0.copy()
    return orc.lora_apply_rows(_bits(x), uor, sor, Au, Bu, y, threads)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_dense_merged_weight_bruteforce(seed):
    rng = np.random.default_rng(seed)
    E, n_ad = 3, 5
    a, e, A, B, x, s, y0 = _random_problem(rng, E=E, n_ad=n_ad)
    y = _oracle_full(a, e, A, B, x, s, y0, E, n_ad)
    W = rng.standard_normal((x.shape[1], y0.shape[1]))           # base weight
    ref = np.empty(y0.shape, np.float64)
    for i in range(x.shape[0]):
        xi = x[i].astype(np.float64)
        if a[i] < 0:
            ref[i] = y0[i]
            continue
        u = a[i] * E + e[i]
        Wp = W + float(s[a[i]]) * (A[u].astype(np.float64) @ B[u].astype(np.float64))  # P:165 W' = W + AB
        ref[i] = y0[i].astype(np.float64) + (xi @ Wp - xi @ W)
    # oracle rounds once to fp32; the brute force differs only by float64 rounding
    np.testing.assert_allclose(y.astype(np.float64), ref, rtol=2 ** -23, atol=1e-9)
    # rows with a = -1 are bit-identical
    np.testing.assert_array_equal(y[a < 0].view(np.uint32), y0[a < 0].view(np.uint32))


def test_peft_transposed_form():
    """North-star form W + s*B_p*A_p with A_p = A^T (r x h_in), B_p = B^T (h_out x r)."""
    rng = np.random.default_rng(7)
    E, n_ad = 3, 5
    a, e, A, B, x, s, y0 = _random_problem(rng, E=E, n_ad=n_ad)
    y = _oracle_full(a, e, A, B, x, s, y0, E, n_ad)
    Wt = rng.standard_normal((y0.shape[1], x.shape[1]))          # PEFT weight [out, in]
    for i in range(x.shape[0]):
        if a[i] < 0:
            continue
        u = a[i] * E + e[i]
        Ap, Bp = A[u].T.astype(np.float64), B[u].T.astype(np.float64)
        Wp = Wt + float(s[a[i]]) * (Bp @ Ap)
        ref = y0[i] + (Wp @ x[i] - Wt @ x[i])
        np.testing.assert_allclose(y[i], ref, rtol=2 ** -23, atol=1e-9)


# ---------------------------------------------------------------------------
# exact-integer probes (numpy int64 matmul; every partial sum exact)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed,h_in,h_out,r", [(0, 64, 48, 8), (1, 32, 16, 1), (2, 8, 64, 4)])
def test_exact_integer_probes(seed, h_in, h_out, r):
    rng = np.random.default_rng(seed)
    T, n_ad, E = 50, 6, 2
    a = rng.integers(-1, n_ad, T).astype(np.int32)
    e = rng.integers(0, E, T).astype(np.int32)
    Ai = rng.integers(-1, 2, (n_ad * E, h_in, r))
    Bi = rng.integers(-1, 2, (n_ad * E, r, h_out))
    xi = rng.integers(-2, 3, (T, h_in))
    yi = rng.integers(-50, 51, (T, h_out))
    s = np.array([0.5, 1.0, 2.0] * 2, np.float32)
    y = _oracle_full(a, e, Ai.astype(np.float32), Bi.astype(np.float32), xi.astype(np.float32), s,
                     yi.astype(np.float32), E, n_ad)
    exp = yi.astype(np.float64).copy()
    for i in range(T):
        if a[i] >= 0:
            u = a[i] * E + e[i]
            exp[i] += float(s[a[i]]) * ((xi[i] @ Ai[u]) @ Bi[u])      # int64 exact
    np.testing.assert_array_equal(y, exp.astype(np.float32))


def test_rank1_outer_product():
    rng = np.random.default_rng(3)
    h_in, h_out, T = 24, 40, 6
    a_vec = _rand_bf16(rng, (1, h_in, 1), -1, 1, 2 ** -6)
    b_vec = _rand_bf16(rng, (1, 1, h_out), -1, 1, 2 ** -6)
    x = _rand_bf16(rng, (T, h_in))
    ids = np.zeros(T, np.int32)
    y = _oracle_full(ids, ids, a_vec, b_vec, x, np.array([2.0], np.float32),
                     np.zeros((T, h_out), np.float32), 1, 1)
    ref = 2.0 * np.outer(x.astype(np.float64) @ a_vec[0, :, 0], b_vec[0, 0])
    np.testing.assert_allclose(y, ref, rtol=2 ** -23, atol=0)


# ---------------------------------------------------------------------------
# invariants
# ---------------------------------------------------------------------------
def test_no_lora_rows_bit_identical_including_negative_zero():
    rng = np.random.default_rng(4)
    a, e, A, B, x, s, y0 = _random_problem(rng, no_lora=1.0)
    y0[0, 0] = -0.0
    y = _oracle_full(a, e, A, B, x, s, y0, 3, 5)
    np.testing.assert_array_equal(y.view(np.uint32), y0.view(np.uint32))
    yb = _oracle_full(a, e, A, B, x, s, y0, 3, 5, y_bits=True)
    np.testing.assert_array_equal(yb, _bits(y0))


def test_permutation_equivariance_bit_exact():
    rng = np.random.default_rng(5)
    a, e, A, B, x, s, y0 = _random_problem(rng, T=64)
    y = _oracle_full(a, e, A, B, x, s, y0, 3, 5, y_bits=True)
    p = rng.permutation(64)
    yp = _oracle_full(a[p], e[p], A, B, x[p], s, y0[p], 3, 5, y_bits=True)
    np.testing.assert_array_equal(yp, y[p])


def test_linearity_in_scale_and_zero_scale():
    rng = np.random.default_rng(6)
    a, e, A, B, x, s, y0 = _random_problem(rng, no_lora=0.0)
    z = np.zeros_like(y0)
    y1 = _oracle_full(a, e, A, B, x, s, z, 3, 5)
    y2 = _oracle_full(a, e, A, B, x, 2 * s, z, 3, 5)
    np.testing.assert_array_equal(y2, 2 * y1)                   # power-of-two scaling is exact
    y0s = _oracle_full(a, e, A, B, x, 0 * s, y0, 3, 5)
    np.testing.assert_array_equal(y0s, y0)


def test_thread_count_invariance():
    rng = np.random.default_rng(8)
    a, e, A, B, x, s, y0 = _random_problem(rng, T=200, h_in=64, h_out=64, r=8)
    y1 = _oracle_full(a, e, A, B, x, s, y0, 3, 5, threads=1)
    y4 = _oracle_full(a, e, A, B, x, s, y0, 3, 5, threads=4)
    np.testing.assert_array_equal(y1.view(np.uint32), y4.view(np.uint32))


def test_out_of_range_ids_rejected():
    with pytest.raises(ValueError):
        orc.unit_tables(np.array([0, 4]), np.array([0, 0]), 2, 4, np.ones(4))
    with pytest.raises(ValueError):
        orc.unit_tables(np.array([0, -2]), np.array([0, 0]), 2, 4, np.ones(4))
    with pytest.raises(ValueError):
        orc.unit_tables(np.array([0, 1]), np.array([0, 2]), 2, 4, np.ones(4))


# ---------------------------------------------------------------------------
# segmentation (a1)
# ---------------------------------------------------------------------------
def _segment_bruteforce(a, e, E):
    rows = [(int(a[i]) * E + (0 if e is None else int(e[i])), i) for i in range(len(a)) if a[i] >= 0]
    rows = sorted(rows)                                   # (key, original index)
    perm = [i for _, i in rows]
    offs, keys, pos = [0], [], 0
    for k, grp in itertools.groupby(rows, key=lambda t: t[0]):
        pos += len(list(grp))
        offs.append(pos)
        keys.append(k)
    return perm, offs, keys


def test_segment_golden():
    g = json.load(open(os.path.join(GOLDEN, "segment_hand.json")))
    for c in g["cases"]:
        e = None if c["expert_ids"] is None else np.array(c["expert_ids"], np.int32)
        perm, offs, keys = oracle.segment(np.array(c["adapter_ids"], np.int32), e, c["E"])
        assert perm.tolist() == c["perm"], c["name"]
        assert offs.tolist() == c["seg_offsets"], c["name"]
        assert keys.tolist() == c["seg_keys"], c["name"]


@pytest.mark.parametrize("seed", range(6))
def test_segment_vs_bruteforce(seed):
    rng = np.random.default_rng(seed)
    T = int(rng.integers(0, 300))
    n_ad, E = int(rng.integers(1, 40)), int(rng.integers(1, 9))
    a = rng.integers(-1, n_ad, T).astype(np.int32)
    e = rng.integers(0, E, T).astype(np.int32)
    perm, offs, keys = oracle.segment(a, e, E)
    bp, bo, bk = _segment_bruteforce(a, e, E)
    assert perm.tolist() == bp and offs.tolist() == bo and keys.tolist() == bk


# ---------------------------------------------------------------------------
# geometry and generator pins
# ---------------------------------------------------------------------------
def test_mixtral_adapter_geometry_matches_paper():
    """1.69 GB per Mixtral adapter at rank 64: separate gate/up/down."""
    cfg = li.CONFIGS["mixtral_decode"]
    per_layer = sum((s.h_in + s.h_out) * cfg.rank * 2 * s.n_experts for s in cfg.slots)
    total = per_layer * 32
    assert total == int(1.6875 * 2 ** 30)
    assert abs(total / 2 ** 30 - 1.69) < 0.005


def test_splitmix64_known_answer():
    # splitmix64 reference: state 0, first output = mix64(0x9E3779B97F4A7C15)
    assert int(li.mix64(np.uint64(0x9E3779B97F4A7C15))) == 0xE220A8397B1DCDAF
    assert int(li.mix64(np.uint64(2 * 0x9E3779B97F4A7C15 % 2 ** 64))) == 0x6E789E6AA1B965F4


def test_generated_values_exact_and_bounded():
    bits = li.unit_A_bits(7, 0, 3, 256, 8)
    f = li.bf16_bits_to_f32(bits)
    q = f * 2.0 ** li.shift_A(256)
    assert np.all(q == np.round(q)) and q.min() >= -128 and q.max() <= 127
    assert abs(f.std() * np.sqrt(256) - 0.577) < 0.2


def test_c_generator_matches_numpy_generator():
    units = np.array([0, 5, 4095, 123456], np.uint64)
    A = li.units_A_bits(77, 2, units, 192, 16)
    Bm = li.units_B_bits(77, 2, units, 16, 320)
    for i, u in enumerate(units):
        np.testing.assert_array_equal(A[i], li.unit_A_bits(77, 2, int(u), 192, 16))
        np.testing.assert_array_equal(Bm[i], li.unit_B_bits(77, 2, int(u), 16, 320))
    rows = np.array([3, 0, 999999])
    np.testing.assert_array_equal(li.gen_rows_fast(5, li.tag_of(li.KIND_X, 1), rows, 256, li.shift_x()),
                                  li.x_rows_bits(5, 1, rows, 256))


def test_zipf_and_experts():
    cfg = li.CONFIGS["mixtral_decode"]
    b = li.make_batch(li.with_tokens(cfg, 20000))
    p = li.zipf_probs(cfg.n_adapters)
    tok = b.adapter_ids[::2]
    freq = np.bincount(tok, minlength=cfg.n_adapters) / tok.size
    assert abs(freq[0] - p[0]) < 0.02 and abs(freq[1] - p[1]) < 0.015
    ex = b.expert_ids.reshape(-1, 2)
    assert np.all(ex[:, 0] != ex[:, 1]) and ex.min() >= 0 and ex.max() < 8


def test_apply_slot_tiny_runs():
    cfg = li.CONFIGS["tiny"]
    b = li.make_batch(cfg)
    y = oracle.apply_slot(cfg, 0, b)
    assert y.shape == (64, 256) and np.isfinite(y).all()


@pytest.mark.parametrize("world,n_hot,ep", [(1, 0, False), (2, 0, False), (3, 2, False), (4, 5, False),
                                            (2, 0, True), (3, 0, True)])
def test_shard_dispatch_pins(world, n_hot, ep):
    """shard_dispatch / owner_of against a per-row brute force of the routing
    rule (R19) and its invariants: the exchanged rows and
    the rows kept in place partition every rank's valid rows, the count matrix
    has a zero diagonal and matches the row lists, replicated adapters never
    leave their source, and a single rank exchanges nothing."""
    import lora_inputs as li
    cfg = li.Config("pin_shard", 13, (li.Slot("s", 64, 64, 4, 0),), 8, 12, 4, 2, 41, "fp32", no_lora_frac=0.1)
    b = li.make_batch(cfg)
    k = b.top_k
    disp = orc.shard_dispatch(b, world, n_hot, ep)
    src = np.empty(b.n_rows, np.int64)
    for g in range(world):
        t0, t1 = (cfg.n_tokens * g) // world, (cfg.n_tokens * (g + 1)) // world
        src[t0 * k:t1 * k] = g
    # brute force, one row at a time
    exp_recv = {d: [] for d in range(world)}
    exp_local = {d: [] for d in range(world)}
    for s_ in range(world):
        for i in range(b.n_rows):
            if src[i] != s_ or b.adapter_ids[i] < 0:
                continue
            a = int(b.adapter_ids[i])
            if ep:
                o = int(b.expert_ids[i]) % world
            else:
                o = s_ if a < n_hot else (a - n_hot) % world
            (exp_local if o == s_ else exp_recv)[o].append(i)
    for d in range(world):
        np.testing.assert_array_equal(disp[d]["rows"], np.array(exp_recv[d], np.int64))
        np.testing.assert_array_equal(disp[d]["local"], np.array(exp_local[d], np.int64))
    counts = disp[0]["counts"]
    assert np.all(np.diag(counts) == 0)
    for d in range(world):
        assert counts[:, d].sum() == len(disp[d]["rows"])
    valid = b.adapter_ids >= 0
    for s_ in range(world):
        n_valid_s = int(np.sum(valid & (src == s_)))
        assert counts[s_].sum() + len(disp[s_]["local"]) == n_valid_s
    if not ep:
        hot_moved = [i for d in range(world) for i in disp[d]["rows"] if b.adapter_ids[i] < n_hot]
        assert hot_moved == []
    if world == 1:
        assert len(disp[0]["rows"]) == 0


def test_shard_dispatch_golden_hand_cases():
    """shard_dispatch against hand-worked routing cases (tests/golden/shard_hand.json,
    P:288-291 / P:323-335 with DESIGN.md R18/R19), independent of owner_of's code."""
    g = json.load(open(os.path.join(GOLDEN, "shard_hand.json")))
    for c in g["cases"]:
        a = np.array(c["adapter_ids"], np.int32)
        e = np.array(c["expert_ids"], np.int32)
        k = c["top_k"]
        b = li.Batch(a, e, a.size // k, k)
        disp = orc.shard_dispatch(b, c["world"], c["n_hot"], c["ep"], c.get("pp", 1), c.get("layer", 0))
        for d in range(c["world"]):
            assert disp[d]["rows"].tolist() == c["rows"][d], (c["name"], d)
            assert disp[d]["local"].tolist() == c["local"][d], (c["name"], d)
        assert disp[0]["counts"].tolist() == c["counts"], c["name"]


# ---------------------------------------------------------------------------
# fp64 -> bf16 rounding of values between float32 grid points (one rounding,
# not fp64 -> fp32 -> bf16): hand cases
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("d,bits", [
    (1.0 + 2 ** -8 + 2 ** -40, 0x3F81),        # just above the tie 1 + 2^-8 -> up
    (1.0 + 2 ** -8 - 2 ** -40, 0x3F80),        # just below -> down
    (1.0 + 3 * 2 ** -8 - 2 ** -40, 0x3F81),    # just below the tie between 0x3F81 / 0x3F82
    (1.0 + 3 * 2 ** -8 + 2 ** -40, 0x3F82),
    (-(1.0 + 2 ** -8 + 2 ** -40), 0xBF81),
    (2.0 ** -133, 0x0001),                     # smallest bf16 subnormal
    (2.0 ** -134, 0x0000),                     # tie between 0 and 2^-133 -> even (0)
    (2.0 ** -134 + 2.0 ** -160, 0x0001),       # above that tie
    (3 * 2.0 ** -134, 0x0002),                 # tie between 1 and 2 quanta -> even
    ((2 - 2 ** -8) * 2.0 ** 127, 0x7F80),      # tie between max finite and 2^128 -> even -> inf
    ((2 - 2 ** -8) * 2.0 ** 127 * (1 - 2 ** -40), 0x7F7F),
    (0.1, 0x3DCD),                             # 0.1 = 0x3DCCCCCD in fp32; bf16 RNE -> 0x3DCD
])
def test_bf16_rounding_between_float32_grid_points(d, bits):
    assert orc.round_bf16(d) == bits


# ---------------------------------------------------------------------------
# apply_slot / prepare_slot glue: row -> unit -> regenerated weights, x rows,
# y0 rows, scale; pinned against a dense per-row brute force built from the
# numpy (not C) generator and float64 numpy arithmetic
# ---------------------------------------------------------------------------
def _apply_slot_bruteforce(cfg, slot_index, batch, rows, y0):
    sl = cfg.slots[slot_index]
    s = cfg.scale()
    x = li.bf16_bits_to_f32(li.x_rows_bits(cfg.seed, sl.xbuf, rows, sl.h_in)).astype(np.float64)
    if y0 == "random":
        y = li.bf16_bits_to_f32(li.y0_rows_bits(cfg.seed, slot_index, rows, sl.h_out)).astype(np.float64)
    else:
        y = np.zeros((len(rows), sl.h_out))
    for n, i in enumerate(rows):
        a = int(batch.adapter_ids[i])
        if a < 0:
            continue
        u = a * sl.n_experts + int(batch.expert_ids[i])
        A = li.bf16_bits_to_f32(li.unit_A_bits(cfg.seed, slot_index, u, sl.h_in, cfg.rank)).astype(np.float64)
        Bm = li.bf16_bits_to_f32(li.unit_B_bits(cfg.seed, slot_index, u, cfg.rank, sl.h_out)).astype(np.float64)
        W = np.random.default_rng(n).standard_normal((sl.h_in, sl.h_out))  # base weight (P:165 W' = W + AB)
        y[n] += x[n] @ (W + float(s[a]) * (A @ Bm)) - x[n] @ W
    return y


@pytest.mark.parametrize("name,y0", [("tiny", "random"), ("tiny", "zero"), ("tiny_dense", "random"), ("mid", "random")])
def test_apply_slot_against_dense_bruteforce(name, y0):
    if name == "mid":
        cfg = li.Config("mid", 8, (li.Slot("a", 128, 192, 4, 0), li.Slot("b", 192, 128, 4, 1)), 16, 24, 4, 2,
                        60, "bf16")
    else:
        cfg = li.CONFIGS[name]
    b = li.make_batch(cfg)
    for si in range(len(cfg.slots)):
        got = orc.apply_slot(cfg, si, b, y0=y0)
        ref = _apply_slot_bruteforce(cfg, si, b, np.arange(b.n_rows), y0)
        if cfg.y_dtype == "fp32":
            np.testing.assert_allclose(got.astype(np.float64), ref, rtol=2 ** -23, atol=1e-12)
        else:  # one bf16 rounding of the exact value: within half an ulp (2^-9 relative)
            np.testing.assert_allclose(li.bf16_bits_to_f32(got).astype(np.float64), ref, rtol=2 ** -8, atol=1e-30)
        # rows without a LoRA are exactly y0
        none = np.flatnonzero(b.adapter_ids < 0)
        if none.size:
            np.testing.assert_array_equal(np.asarray(got)[none].astype(np.float64) if cfg.y_dtype == "fp32"
                                          else li.bf16_bits_to_f32(got[none]).astype(np.float64), ref[none])


def test_apply_slot_all_rows_equals_apply_slot():
    cfg = li.Config("mid", 8, (li.Slot("a", 128, 192, 4, 0),), 16, 24, 4, 2, 90, "bf16", no_lora_frac=0.1)
    b = li.make_batch(cfg)
    for y0 in ("random", "zero"):
        full = orc.apply_slot(cfg, 0, b, y0=y0)
        chunked = orc.apply_slot_all_rows(cfg, 0, b, y0=y0, unit_chunk=3)
        np.testing.assert_array_equal(full, chunked)
