"""Host-side placement policy (paper_2604_07173_b200/placement.py; R19)."""
import numpy as np

import lora_inputs as li
from oracle import oracle as orc
from paper_2604_07173_b200 import placement as P


def test_owner_matches_oracle_routing():
    cfg = li.CONFIGS["mixtral_sharded"]
    b = li.make_batch(cfg)
    for G in (2, 3, 8):
        src = P.sources_of_rows(cfg.n_tokens, cfg.top_k, G)
        for h in (0, 1, 5, 64):
            np.testing.assert_array_equal(P.owner(b.adapter_ids, G, h, src),
                                          orc.owner_of(b.adapter_ids, G, h, src))
        np.testing.assert_array_equal(P.owner(b.adapter_ids, G, 0, src), orc.owner_of(b.adapter_ids, G))


def test_rank_costs_brute_force():
    rng = np.random.default_rng(5)
    a = rng.integers(-1, 12, 200)
    e = rng.integers(0, 3, 200)
    G, h = 3, 2
    src = np.repeat(np.arange(G), [70, 60, 70])
    U, R, X = 1000.0, 10.0, 7.0
    got = P.rank_costs(a, e, src, G, h, U, R, X, hbm_gbs=1.0, link_gbs=1.0) * 1e9
    for g in range(G):
        units, mine, rin, rout = set(), 0, 0, 0
        for i in range(200):
            if a[i] < 0:
                continue
            o = int(src[i]) if a[i] < h else (a[i] - h) % G
            if o == g:
                units.add((a[i], e[i]))
                mine += 1
                rin += src[i] != g
            elif src[i] == g:
                rout += 1
        assert abs(got[g] - (len(units) * U + (mine + rout) * R + max(rin, rout) * X)) < 1e-6


def test_choose_replicates_a_dominant_adapter():
    T = 4096
    a = np.zeros(T, np.int64)                # every row on adapter 0
    a[::64] = np.arange(T // 64) % 40 + 1    # a thin tail
    src = P.sources_of_rows(T, 1, 4)
    r = P.choose_n_replicated(a, None, src, 4, unit_bytes=1e6, row_bytes=1e5, xfer_bytes=1e5)
    assert r["n_replicated"] >= 1 and r["table"][r["n_replicated"]] < r["table"][0]
    assert P.choose_n_replicated(a, None, src[:0] * 0, 1, 1.0, 1.0, 1.0)["n_replicated"] == 0


def test_slot_bytes_mixtral():
    u, r, x = P.slot_bytes([4096, 4096, 14336], [14336, 14336, 4096], [0, 0, 1], 64, 2, 4)
    assert u == 2 * 64 * 3 * (4096 + 14336)
    assert r == 2 * 4096 + 2 * 14336 + 2 * 2 * (14336 * 2 + 4096)
    assert x == 2 * 4096 + 2 * 14336 + 4 * (14336 * 2 + 4096)


def test_rank_hbm_bytes_brute_force():
    """Per-rank algorithmic bytes of a sharded apply (bench.py's sharded
    roofline): touched units once, served rows once, own rows served
    elsewhere accumulated once -- per-row brute force, DP with replication
    and expert parallel."""
    rng = np.random.default_rng(9)
    n = 300
    a = rng.integers(-1, 16, n)
    e = rng.integers(0, 4, n)
    G = 4
    src = np.repeat(np.arange(G), n // G)
    U, R = 500.0, 3.0
    for h, ep in ((0, False), (3, False), (0, True)):
        got = P.rank_hbm_bytes(a, e, src, G, h, U, R, ep=ep)
        for g in range(G):
            units, mine, rout = set(), 0, 0
            for i in range(n):
                if a[i] < 0:
                    continue
                if ep:
                    o = int(e[i]) % G
                else:
                    o = int(src[i]) if a[i] < h else (a[i] - h) % G
                if o == g:
                    units.add((a[i], e[i]))
                    mine += 1
                elif src[i] == g:
                    rout += 1
            assert abs(got[g] - (len(units) * U + (mine + rout) * R)) < 1e-6, (h, ep, g)


def test_rank_costs_push_brute_force():
    """Push-path model: a row's x read and y RMW land on its SOURCE's HBM,
    owners pay the units they serve; link bytes in/out per rank; per-row
    brute force for DP with replication, EP and hybrid EP_x-PP_y."""
    rng = np.random.default_rng(6)
    n = 240
    a = rng.integers(-1, 12, n)
    e = rng.integers(0, 4, n)
    G = 4
    src = np.repeat(np.arange(G), n // G)
    U, R, X, D = 1000.0, 10.0, 7.0, 3.0
    for h, ep, pp, layer in ((0, False, 1, 0), (2, False, 1, 0), (0, True, 1, 0), (0, True, 2, 1), (0, True, 2, 0)):
        got = P.rank_costs_push(a, e, src, G, h, U, R, X, D, hbm_gbs=1.0, link_gbs=1.0, fixed_s=0.0, ep=ep, pp=pp,
                                layer=layer) * 1e9
        for g in range(G):
            units, own_rows, rin, rout = set(), 0, 0, 0
            for i in range(n):
                if a[i] < 0:
                    continue
                if ep:
                    x = G // pp
                    o = (layer % pp) * x + int(e[i]) % x
                else:
                    o = int(src[i]) if a[i] < h else (a[i] - h) % G
                if src[i] == g:
                    own_rows += 1
                if o == g:
                    units.add((a[i], e[i]))
                    rin += src[i] != g
                elif src[i] == g:
                    rout += 1
            hbm = len(units) * U + own_rows * R
            link = max(rin * X + rout * D, rout * X + rin * D)
            assert abs(got[g] - max(hbm, link)) < 1e-6, (h, ep, pp, g)


def test_hybrid_owner_matches_oracle_routing():
    b = li.make_batch(li.CONFIGS["mixtral_decode"])
    for y in (1, 2, 4, 8):
        for layer in (0, 1, 5):
            x = 8 // y
            own = np.where(b.adapter_ids >= 0, (layer % y) * x + b.expert_ids % x, -1)
            np.testing.assert_array_equal(own, orc.owner_of(b.adapter_ids, 8, 0, None, b.expert_ids, True, y, layer))


def test_push_model_predicts_config5_efficiency():
    """The push-path model (registered buffers, transfers fused into the
    kernels) at G = 8 on config 5 -- the design target of >= 0.70 strong-
    scaling efficiency (north star)."""
    cfg = li.CONFIGS["mixtral_sharded"]
    b = li.make_batch(cfg)
    u, r, x, d = P.slot_bytes_push([s.h_in for s in cfg.slots], [s.h_out for s in cfg.slots],
                                   [s.xbuf for s in cfg.slots], 64, 2, 2)
    t1 = P.rank_costs_push(b.adapter_ids, b.expert_ids, np.zeros(b.n_rows, int), 1, 0, u, r, x, d, fixed_s=0)[0]
    for G in (2, 4, 8):
        src = P.sources_of_rows(cfg.n_tokens, 2, G)
        ch = P.choose_placement(b.adapter_ids, b.expert_ids, src, G, u, r, 0.0, x_bytes=x, d_bytes=d)
        tg = min(ch["table"].values())
        assert t1 / (G * tg) >= 0.70, (G, t1 / (G * tg))


def test_bench_algorithmic_dispatch_rule(monkeypatch):
    """bench.algorithmic attributes a slot's bytes to the tcgen05 kernels
    exactly as the library dispatches: segments of more than small_max rows,
    tcgen05 ranks 8-128, and only when those segments hold at least
    LORA_TC_MIN_ROWS rows together (256, 2048 at r <= 16); hand-built batch."""
    import bench
    import lora_inputs as li
    monkeypatch.delenv("LORA_TC_MIN_ROWS", raising=False)
    # 300 rows of adapter 0 (one 300-row segment), 5 singletons
    a = np.array([0] * 300 + [1, 2, 3, 4, 5], np.int32)
    batch = li.Batch(a, np.zeros_like(a), a.size, 1)
    for r, tc in ((64, True), (32, True), (128, True), (8, False), (16, False)):
        cfg = li.Config("t", 1, (li.Slot("s", 256, 512, 1, 0),), r, 8, 1, 1, a.size, "bf16")
        out = bench.algorithmic(cfg, batch, [0])
        big_rows = 300
        if tc:  # the big segment on tcgen05: its unit's A/B, rows' x and y
            assert out["tc05_shrink"] == 256 * r * 2 + big_rows * 256 * 2
            assert out["tc05_expand"] == 512 * r * 2 + big_rows * 512 * 2 * 2
            assert out["simt_shrink"] == 5 * 256 * r * 2 + 5 * 256 * 2
        else:  # r <= 16: 300 < 2048 rows in large segments -> CUDA cores only
            assert out["tc05_shrink"] == 0 and out["tc05_expand"] == 0
            assert out["simt_shrink"] == 6 * 256 * r * 2 + 305 * 256 * 2
    monkeypatch.setenv("LORA_TC_MIN_ROWS", "0")
    cfg = li.Config("t", 1, (li.Slot("s", 256, 512, 1, 0),), 16, 8, 1, 1, a.size, "bf16")
    assert bench.algorithmic(cfg, batch, [0])["tc05_shrink"] > 0
    monkeypatch.setenv("LORA_TC_MIN_ROWS", "400")
    cfg = li.Config("t", 1, (li.Slot("s", 256, 512, 1, 0),), 64, 8, 1, 1, a.size, "bf16")
    assert bench.algorithmic(cfg, batch, [0])["tc05_shrink"] == 0
