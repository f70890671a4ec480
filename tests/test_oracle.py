"""CPU suite for the oracle: SPEC.md worked examples, golden vectors from the compiled reference,
and (where oracle/_ref exists) restatement == reference on fresh random inputs."""
import hashlib
import tempfile
from pathlib import Path

import numpy as np
import pytest

from paper_1805_08995_b200.api import FamilyParams, MatchConfig
from paper_1805_08995_b200.synth import make_dataset


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def both(restatement, request):
    import oracle_lib
    ref = oracle_lib.reference()
    return [restatement] + ([ref] if ref is not None else [])


# ---- SPEC.md worked examples (known answers) -----------------------------------------------------
def test_reduce_dot_examples(restatement, request):
    for orc in both(restatement, request):
        ones = np.ones(128)
        e0 = np.zeros(128)
        e0[0] = 1
        b = np.arange(128, dtype=np.float64) + 0.5
        for rr in range(8):
            assert orc.reduce_dot(ones, ones, rr) == 128.0
            assert orc.reduce_dot(e0, b, rr) == b[0]
        rng = np.random.default_rng(0)
        a, c = rng.normal(size=128), rng.normal(size=128)
        exact = float(np.sum(a.astype(np.longdouble) * c.astype(np.longdouble)))
        for rr in range(8):
            assert abs(orc.reduce_dot(a, c, rr) - exact) <= 128 * np.finfo(np.float64).eps * np.sum(np.abs(a * c))
        with pytest.raises(ValueError):
            orc.reduce_dot(a, c, 8)


def test_reduce_dot_order_is_tree_then_serial(restatement):
    # an input where summation order changes the fp64 result pins the DAG itself
    rng = np.random.default_rng(1)
    a = rng.normal(size=128) * 10.0 ** rng.integers(-8, 8, size=128)
    b = rng.normal(size=128)
    p = a * b

    def model(rr):
        s = p.copy()
        w = 128
        while w > (1 << rr):
            w //= 2
            s[:w] = s[:w] + s[w:2 * w]
        acc = s[0]
        for i in range(1, w):
            acc = acc + s[i]
        return acc

    vals = {rr: restatement.reduce_dot(a, b, rr) for rr in range(8)}
    assert len(set(vals.values())) > 1, "test vector must be order sensitive"
    for rr in range(8):
        assert vals[rr] == model(rr)


def test_family_examples(restatement, request):
    for orc in both(restatement, request):
        p = FamilyParams()
        sp, lp = orc.build_family(p)
        assert sp.shape == (48, 128) and lp.shape == (128, 128)
        sp2, lp2 = orc.build_family(p)
        assert np.array_equal(sp, sp2) and np.array_equal(lp, lp2)
        sp3, _ = orc.build_family(FamilyParams(seed=2))
        assert not np.array_equal(sp, sp3)
        assert np.isfinite(sp).all() and np.isfinite(lp).all()
        # long planes come from a sentinel stream: independent of table_count (hashing.cpp:17-19)
        _, lp4 = orc.build_family(FamilyParams(table_count=3))
        assert np.array_equal(lp, lp4)
        for bad in (FamilyParams(short_bits=0), FamilyParams(short_bits=33), FamilyParams(long_bits=8),
                    FamilyParams(long_bits=129), FamilyParams(table_count=0)):
            with pytest.raises(ValueError):
                orc.build_family(bad)


def test_centering_examples(restatement, request):
    for orc in both(restatement, request):
        v = np.arange(128, dtype=np.uint8)
        assert np.array_equal(orc.centering([v]), v.astype(np.float64))
        two = np.stack([np.zeros(128, np.uint8), np.full(128, 2, np.uint8)])
        assert np.array_equal(orc.centering([two]), np.ones(128))
        rng = np.random.default_rng(3)
        d = rng.integers(0, 256, size=(1000, 128), dtype=np.uint8)
        want = d.astype(np.uint64).sum(0).astype(np.float64) / 1000.0
        assert np.array_equal(orc.centering([d[:400], d[400:]]), want)
        with pytest.raises(ValueError):
            orc.centering([])


def test_code_examples(restatement, request):
    for orc in both(restatement, request):
        p = FamilyParams()
        sp, lp = orc.build_family(p)
        c = np.full(128, 77.0)
        s, l = orc.compute_codes(p, sp, lp, c, np.full((1, 128), 77, np.uint8))
        assert not s.any() and not l.any()                          # ties -> 0
        # naive per-component sign computation away from ties
        rng = np.random.default_rng(5)
        d = rng.integers(0, 256, size=(64, 128), dtype=np.uint8)
        cen = orc.centering([d])
        s, l = orc.compute_codes(p, sp, lp, cen, d)
        cd = d.astype(np.float64) - cen
        dots_s = cd @ sp.T
        dots_l = cd @ lp.T
        safe_s = np.abs(dots_s) > 1e-6
        bits_s = (s[:, :, None] >> np.arange(8)[None, None, :]) & 1
        assert np.array_equal(bits_s.reshape(64, 48)[safe_s], (dots_s > 0)[safe_s])
        bits_l = ((l[:, :, None] >> np.arange(64, dtype=np.uint64)[None, None, :]) & np.uint64(1)).reshape(64, 128)
        safe_l = np.abs(dots_l) > 1e-6
        assert np.array_equal(bits_l[safe_l].astype(bool), (dots_l > 0)[safe_l])
        assert (s < 256).all()
        # centering unset -> logic_error (hashing.cpp:131-132)
        with pytest.raises(RuntimeError):
            orc.compute_codes(p, sp, lp, None, d)


def test_bucket_and_lookup_examples(restatement, request):
    for orc in both(restatement, request):
        m, L = 8, 6
        offs, pts = orc.build_bucket_index(m, L, np.zeros((0, L), np.uint32))
        assert not offs.any()
        same = np.tile(np.array([[3, 1, 4, 1, 5, 9]], np.uint32), (2, 1))
        offs, pts = orc.build_bucket_index(m, L, same)
        for t in range(L):
            c = same[0, t]
            assert pts[t, offs[t, c]:offs[t, c + 1]].tolist() == [0, 1]
        rng = np.random.default_rng(7)
        codes = rng.integers(0, 256, size=(500, L), dtype=np.uint32)
        offs, pts = orc.build_bucket_index(m, L, codes)
        for t in range(L):                                          # SPEC.md:241 reconstruction
            assert sorted(pts[t].tolist()) == list(range(500))
            for c in range(256):
                b = pts[t, offs[t, c]:offs[t, c + 1]]
                assert (codes[b, t] == c).all() and (np.diff(b.astype(np.int64)) > 0).all()
        q = codes[17].copy()
        cand = orc.lookup_candidates(m, L, q, codes)
        want = np.nonzero((codes == q[None, :]).any(1))[0]
        assert np.array_equal(cand, want) and 17 in cand            # SPEC.md:249 dedup
        assert len(orc.lookup_candidates(m, L, np.full(L, 300, np.uint32), codes)) == 0


def _mk_codes(n, L=6):
    return np.zeros((n, L), np.uint32), np.zeros((n, 2), np.uint64)


def test_rank_and_verify_examples(restatement, request):
    """SPEC.md:257-259 (ranking) and :266-268 (verify) through match_pair on crafted inputs."""
    for orc in both(restatement, request):
        p = FamilyParams()
        # one query, four train points in the same bucket with Hamming distances [5, 3, 40, 41]
        si, li = _mk_codes(1)
        sj, lj = _mk_codes(4)
        for idx, d in enumerate([5, 3, 40, 41]):
            lj[idx, 0] = (1 << d) - 1
        dq = np.zeros((1, 128), np.uint8)
        dt = np.zeros((4, 128), np.uint8)
        dt[0, 0] = 100   # d^2 = 10000
        dt[1, 0] = 10    # d^2 = 100
        dt[2, 0] = 200
        dt[3, 0] = 1     # would win if the 41 were not discarded
        cfg = MatchConfig(top_k=2, hamming_threshold=40)
        rec, st, ranked, rc = orc.match_pair(p, cfg, dq, si, li, dt, sj, lj, want_ranked=True)
        assert rc[0] == 2 and ranked[0].tolist() == [1, 0]          # distances 3 and 5
        assert rec.tolist() == [(0, 1, 100.0)]                      # 100/10000 < 0.64
        # all candidates beyond tau -> empty ranking, no match, no fallback
        cfg0 = MatchConfig(top_k=2, hamming_threshold=2)
        rec, st, ranked, rc = orc.match_pair(p, cfg0, dq, si, li, dt, sj, lj, want_ranked=True)
        assert rc[0] == 0 and len(rec) == 0 and st["fallback_queries"] == 0
        # tau = n, k = |candidates| -> full sort by (distance, index)
        cfgf = MatchConfig(top_k=4, hamming_threshold=128)
        _, _, ranked, rc = orc.match_pair(p, cfgf, dq, si, li, dt, sj, lj, want_ranked=True)
        assert rc[0] == 4 and ranked[0].tolist() == [1, 0, 2, 3]
        # single ranked candidate -> re-rank fallback keeps the second distance (matcher.cpp:179-189)
        cfg1 = MatchConfig(top_k=10, hamming_threshold=3)
        rec, st, ranked, rc = orc.match_pair(p, cfg1, dq, si, li, dt, sj, lj, want_ranked=True)
        assert st["fallback_queries"] == 1 and rc[0] == 4 and ranked[0, :4].tolist() == [1, 0, 2, 3]
        assert rec.tolist() == [(0, 3, 1.0)]
        # only one candidate at all -> ratio undecidable
        rec, _ = orc.match_pair(p, MatchConfig(), dq, si, li, dt[:1], sj[:1], lj[:1])
        assert len(rec) == 0
        # exact duplicates: second distance 0 -> rejection
        dup = np.zeros((2, 128), np.uint8)
        rec, _ = orc.match_pair(p, MatchConfig(), dq, si, li, dup, *_mk_codes(2))
        assert len(rec) == 0
        # empty train / query sets
        rec, _ = orc.match_pair(p, MatchConfig(), dq, si, li, dt[:0], sj[:0], lj[:0])
        assert len(rec) == 0
        rec, _ = orc.match_pair(p, MatchConfig(), dq[:0], si[:0], li[:0], dt, sj, lj)
        assert len(rec) == 0
        for bad in (MatchConfig(top_k=1), MatchConfig(hamming_threshold=129), MatchConfig(ratio=1.0),
                    MatchConfig(ratio=0.0), MatchConfig(reduce_rounds=8)):
            with pytest.raises(ValueError):
                orc.match_pair(p, bad, dq, si, li, dt, sj, lj)


def test_brute_force_examples(restatement, request):
    for orc in both(restatement, request):
        a = np.zeros((1, 128), np.uint8)
        b = np.full((1, 128), 200, np.uint8)
        assert len(orc.brute_force_match(a, b, 0.8)) == 0
        oh = np.zeros((3, 128), np.uint8)
        oh[0, 0], oh[1, 1], oh[2, 2] = 10, 100, 200
        q = np.zeros((1, 128), np.uint8)
        q[0, 0] = 12
        rec = orc.brute_force_match(q, oh, 0.8)
        assert rec.tolist() == [(0, 0, 4.0)]


# ---- golden vectors from the compiled reference ---------------------------------------------------
def test_restatement_matches_golden_family(restatement, golden):
    g = golden["family"]
    for tag, params in {"default": FamilyParams(), "m10_n96_L4_s99": FamilyParams(10, 96, 4, 99)}.items():
        sp, lp = restatement.build_family(params)
        assert sha(sp) == str(g[tag + "_short_sha"]) and sha(lp) == str(g[tag + "_long_sha"])
        assert np.array_equal(sp[:2, :4], g[tag + "_short_head"])
        assert np.array_equal(lp[-1, -4:], g[tag + "_long_tail"])
    assert restatement.mix64(1, 2, 3) == int(g["mix64_1_2_3"])
    assert restatement.mix64(1, 0xffffffff, 5) == int(g["mix64_seed1_long_5"])


GOLDEN_CFGS = {
    "default": MatchConfig(),
    "tau128": MatchConfig(hamming_threshold=128),
    "k2_min5": MatchConfig(top_k=2, min_candidates_for_ratio=5),
    "tau60_k32_r09": MatchConfig(top_k=32, hamming_threshold=60, ratio=0.9),
    "tau0": MatchConfig(hamming_threshold=0),
}


def test_restatement_matches_golden_dataset(restatement, golden):
    g = golden["small_dataset"]
    params = FamilyParams()
    sp, lp = restatement.build_family(params)
    desc = g["desc"]
    assert np.array_equal(desc, make_dataset(3, 300, seed=11)), "synthetic generator drifted from the fixture"
    cen = restatement.centering([desc[0], desc[1], desc[2]])
    assert np.array_equal(cen, g["centering"])
    codes = []
    for i in range(3):
        s, l = restatement.compute_codes(params, sp, lp, cen, desc[i], 3)
        assert np.array_equal(s, g[f"shorts{i}"]) and np.array_equal(l, g[f"longs{i}"])
        codes.append((s, l))
        for rr in (0, 7):
            s2, l2 = restatement.compute_codes(params, sp, lp, cen, desc[i], rr)
            assert sha(s2) == str(g[f"shorts{i}_rr{rr}_sha"]) and sha(l2) == str(g[f"longs{i}_rr{rr}_sha"])
    offs, pts = restatement.build_bucket_index(8, 6, codes[1][0])
    assert np.array_equal(offs, g["offs1"]) and np.array_equal(pts, g["pts1"])
    for tag, cfg in GOLDEN_CFGS.items():
        for (a, b) in ((0, 1), (1, 2), (2, 0)):
            rec, stats, ranked, rc = restatement.match_pair(params, cfg, desc[a], *codes[a], desc[b], *codes[b],
                                                            want_ranked=True)
            assert np.array_equal(rec, g[f"rec_{tag}_{a}{b}"]), (tag, a, b)
            assert np.array_equal(rc, g[f"rcount_{tag}_{a}{b}"])
            gr = g[f"ranked_{tag}_{a}{b}"]
            for q in range(len(rc)):
                assert np.array_equal(ranked[q, :rc[q]], gr[q, :rc[q]])
            assert list(stats.values()) == g[f"stats_{tag}_{a}{b}"].tolist()
    assert len(g["rec_default_01"]) > 50, "fixture must exercise real matches"
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "m.txt"
        restatement.save_matches("img_a", "img_b", g["rec_default_01"], p)
        assert p.read_bytes() == g["match_text_default_01"].tobytes()
    assert np.array_equal(restatement.brute_force_match(desc[0], desc[1], 0.8), g["brute_01"])


def test_restatement_matches_golden_plans(restatement, golden):
    g = golden["plans"]
    for (k, np_, m) in ((10, 3, 2), (7, 2, 2), (12, 5, 1), (9, 1, 4), (5, 8, 3)):
        pairs, sizes = restatement.plan_exhaustive(k, np_, m)
        assert np.array_equal(pairs, g[f"pairs_{k}_{np_}_{m}"])
        assert np.array_equal(sizes, g[f"sizes_{k}_{np_}_{m}"])
        assert len({(int(a), int(b)) for a, b in pairs}) == k * (k - 1) // 2 and (pairs[:, 0] < pairs[:, 1]).all()


# ---- restatement == compiled reference on fresh inputs (only where oracle/_ref exists) -----------
@pytest.mark.parametrize("params,n,seed", [
    (FamilyParams(), 700, 1), (FamilyParams(8, 128, 6, 5), 1500, 2), (FamilyParams(10, 96, 4, 99), 900, 3),
    (FamilyParams(4, 64, 8, 7), 400, 4), (FamilyParams(12, 128, 2, 3), 1200, 5),
])
def test_restatement_equals_reference_random(restatement, reference, params, n, seed):
    sp, lp = reference.build_family(params)
    sp2, lp2 = restatement.build_family(params)
    assert np.array_equal(sp, sp2) and np.array_equal(lp, lp2)
    shape = "sift" if seed % 2 == 0 else "uniform"
    desc = make_dataset(2, n, seed=100 + seed, shape=shape)
    cen = reference.centering(list(desc))
    assert np.array_equal(cen, restatement.centering(list(desc)))
    codes = []
    for i in range(2):
        for rr in (3, 0, 5, 7):
            a = reference.compute_codes(params, sp, lp, cen, desc[i], rr)
            b = restatement.compute_codes(params, sp, lp, cen, desc[i], rr)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            if rr == 3:
                codes.append(a)
    for cfg in (MatchConfig(), MatchConfig(top_k=5, hamming_threshold=min(50, params.long_bits), ratio=0.7,
                                            min_candidates_for_ratio=4)):
        a = reference.match_pair(params, cfg, desc[0], *codes[0], desc[1], *codes[1], want_ranked=True)
        b = restatement.match_pair(params, cfg, desc[0], *codes[0], desc[1], *codes[1], want_ranked=True)
        assert np.array_equal(a[0], b[0])
        assert a[1] == b[1]
        assert np.array_equal(a[3], b[3])
        for q in range(n):
            assert np.array_equal(a[2][q, :a[3][q]], b[2][q, :b[3][q]])
    if params.short_bits <= 12:
        oa = reference.build_bucket_index(params.short_bits, params.table_count, codes[1][0])
        ob = restatement.build_bucket_index(params.short_bits, params.table_count, codes[1][0])
        assert np.array_equal(oa[0], ob[0]) and np.array_equal(oa[1], ob[1])


def test_list_filter_restatement_equals_reference(restatement, reference):
    """chor_match_pair_lists: match_pair_filtered (matcher.hpp:102-105) with the candidates of every query replaced by a
    given list — thinned, reordered, with repeats.  In oracle/_ref it is the reference's own function; the restatement must
    agree on records, statistics and ranked lists, and unchanged lists must give match_pair."""
    params = FamilyParams()
    sp, lp = reference.build_family(params)
    desc = make_dataset(2, 700, seed=321)
    cen = reference.centering(list(desc))
    codes = [reference.compute_codes(params, sp, lp, cen, desc[i]) for i in range(2)]
    rng = np.random.default_rng(5)
    same_lo, same_ids, lo, ids = [0], [], [0], []
    for q in range(700):
        c = reference.lookup_candidates(params.short_bits, params.table_count, codes[0][0][q], codes[1][0]).tolist()
        same_ids += c
        same_lo.append(len(same_ids))
        kind = q % 4
        if kind == 1:
            c = c[::-1]
        elif kind == 2:
            c = [x for x in c if rng.random() < 0.7] + c[:1]
        elif kind == 3:
            c = []
        ids += c
        lo.append(len(ids))
    for cfg in (MatchConfig(), MatchConfig(top_k=40, hamming_threshold=60), MatchConfig(top_k=3, min_candidates_for_ratio=6)):
        args = (params, cfg, desc[0], *codes[0], desc[1], *codes[1])
        a = reference.match_pair_lists(*args, lo, ids, want_ranked=True)
        b = restatement.match_pair_lists(*args, lo, ids, want_ranked=True)
        assert len(a[0]) > 0 and np.array_equal(a[0], b[0]) and a[1] == b[1] and np.array_equal(a[3], b[3])
        for q in range(700):
            assert np.array_equal(a[2][q, :a[3][q]], b[2][q, :b[3][q]])
        plain = reference.match_pair(*args)
        assert np.array_equal(reference.match_pair_lists(*args, same_lo, same_ids)[0], plain[0])
        assert np.array_equal(restatement.match_pair_lists(*args, same_lo, same_ids)[0], plain[0])


def test_restatement_matches_golden_guided_plans(restatement, golden):
    g = golden["plans_guided"]
    for key in [k for k in g.files if k.startswith("accepted_")]:
        k, np_, m = (int(x) for x in key.split("_")[1:])
        pairs, sizes = restatement.plan_guided(k, np_, m, g[key])
        assert np.array_equal(pairs, g[f"pairs_{k}_{np_}_{m}"]) and np.array_equal(sizes, g[f"sizes_{k}_{np_}_{m}"])
    with pytest.raises(ValueError):
        restatement.plan_guided(10, 3, 2, [(1, 1)])      # self pair
    with pytest.raises(ValueError):
        restatement.plan_guided(10, 3, 2, [(1, 10)])     # unknown image index


def test_guided_plans_equal_reference(restatement, reference):
    rng = np.random.default_rng(4)
    for (k, np_, m) in ((31, 4, 3), (17, 17, 1), (50, 1, 5)):
        acc = rng.integers(0, k, (300, 2)).astype(np.uint32)
        acc = acc[acc[:, 0] != acc[:, 1]]
        a = reference.plan_guided(k, np_, m, acc)
        b = restatement.plan_guided(k, np_, m, acc)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert len(reference.plan_guided(9, 2, 2, np.zeros((0, 2), np.uint32))[0]) == 0


def test_plans_equal_reference(restatement, reference):
    for k in (1, 2, 3, 5, 8, 13, 20, 33):
        for np_ in (1, 2, 3, 5):
            for m in (1, 2, 3, 4):
                a = reference.plan_exhaustive(k, np_, m)
                b = restatement.plan_exhaustive(k, np_, m)
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), (k, np_, m)


def test_guided_restatement_equals_reference(restatement, reference):
    """f4: the band filter around the reference's own match_pair_filtered vs the restatement."""
    import paper_1805_08995_b200 as ch
    from paper_1805_08995_b200.synth import make_dataset
    params, cfg = ch.FamilyParams(), ch.MatchConfig()
    fam = ch.build_hash_family(params)
    d = make_dataset(2, 1200, seed=9)
    rng = np.random.default_rng(1)
    kp = [np.column_stack([np.floor(rng.uniform(0, 1000, 1200)), rng.uniform(0, 800, 1200), np.full(1200, 2.0),
                           np.zeros(1200)]).astype(np.float32) for _ in range(2)]
    cen = reference.centering([d[0], d[1]])
    codes = [reference.compute_codes(params, fam.short_planes, fam.long_planes, cen, d[i]) for i in range(2)]
    base, _ = reference.match_pair(params, cfg, d[0], *codes[0], d[1], *codes[1])
    F = rng.normal(size=(3, 3))
    F[:, 2] *= 300.0
    some_degenerate = np.array([[1.0, 0.0, -7.0], [0.0, 0.0, 0.0], [0.0, 50.0, -20000.0]])
    sizes = []
    for f, band in ((F, 1e9), (F, 150.0), (F, 20.0), (F, 0.0), (np.zeros((3, 3)), 3.0), (some_degenerate, 60.0)):
        a = reference.guided_match_pair(params, cfg, d[0], kp[0], *codes[0], d[1], kp[1], *codes[1], f, band, want_ranked=True)
        b = restatement.guided_match_pair(params, cfg, d[0], kp[0], *codes[0], d[1], kp[1], *codes[1], f, band, want_ranked=True)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]
        assert np.array_equal(a[3], b[3])
        for q in np.flatnonzero(a[3]):
            assert np.array_equal(a[2][q, :a[3][q]], b[2][q, :b[3][q]])
        sizes.append(len(a[0]))
    assert sizes[0] == len(base) == sizes[4] and sizes[3] == 0 and 0 < sizes[1] < sizes[0]


def _band_distances(F, kp_i, kp_j, order):
    """|a x' + b y' + c| / sqrt(a^2 + b^2) for every (query, train point), fp64, one rounding per operation, in the
    operation order of the band filter (geometry.cpp:238-248) with the line's third component associated either way."""
    x, y = kp_i[:, 0].astype(np.float64), kp_i[:, 1].astype(np.float64)
    a = (F[0, 0] * x + F[0, 1] * y) + F[0, 2]
    b = (F[1, 0] * x + F[1, 1] * y) + F[1, 2]
    c = F[2, 0] * x + (F[2, 1] * y + F[2, 2]) if order == 0 else (F[2, 0] * x + F[2, 1] * y) + F[2, 2]
    live = ~((a == 0.0) & (b == 0.0))
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / np.sqrt(a * a + b * b)
        tx, ty = kp_j[:, 0].astype(np.float64), kp_j[:, 1].astype(np.float64)
        d = np.abs((a[:, None] * tx[None, :] + b[:, None] * ty[None, :]) + c[:, None]) * inv[:, None]
    return d, live


def test_guided_line_order_bound(restatement):
    """Row f4 is pinned up to ONE unverifiable fact: the association order of l(2) = F20 x + F21 y + F22 inside
    Eigen's Matrix3d * Vector3d (geometry.cpp:98-101; no Eigen in this image).  This bounds what that fact can change:
    over a fuzz corpus of fundamental matrices, keypoints and bands, (1) count the (query, candidate) decisions that
    differ between the two possible orders and the candidates within 4 ulp of the band edge under either, and (2) run
    the whole guided match under both orders and require identical records, ranked lists and statistics."""
    import paper_1805_08995_b200 as ch
    params, cfg = ch.FamilyParams(), ch.MatchConfig()
    fam = ch.build_hash_family(params)
    decisions = differing = near_edge = moved_c = 0
    try:
        for seed in range(24):
            rng = np.random.default_rng(1000 + seed)
            n = 500
            d = make_dataset(2, n, seed=100 + seed)
            # pixel keypoints the way detectors report them: sub-pixel float32 positions in a ~1000 x 800 image
            kp = [np.column_stack([rng.uniform(0, 1000, n), rng.uniform(0, 800, n), np.full(n, 2.0), np.zeros(n)])
                  .astype(np.float32) for _ in range(2)]
            if seed % 3 == 2:
                F = np.array([[1.0, 0.0, -float(rng.integers(0, 900))], [0.0, 0.0, 0.0], [0.0, 50.0, -20000.0]])
            else:
                F = rng.normal(size=(3, 3))
                F[:, 2] *= 300.0
                if seed % 3 == 1:  # a properly scaled rank-2 matrix (normalize_scale_and_sign leaves |F| = 1)
                    u, sv, vt = np.linalg.svd(F)
                    F = (u * np.array([sv[0], sv[1], 0.0])) @ vt
                    F /= np.linalg.norm(F)
            band = float(rng.choice([0.5, 5.0, 40.0, 150.0, 300.0]))
            d0, live = _band_distances(F, kp[0], kp[1], 0)
            d1, _ = _band_distances(F, kp[0], kp[1], 1)
            d0, d1 = d0[live], d1[live]
            decisions += d0.size
            differing += int(np.count_nonzero((d0 > band) != (d1 > band)))
            edge = 4.0 * np.spacing(band)
            near_edge += int(np.count_nonzero((np.abs(d0 - band) <= edge) | (np.abs(d1 - band) <= edge)))
            moved_c += int(np.count_nonzero(d0 != d1))
            cen = restatement.centering([d[0], d[1]])
            codes = [restatement.compute_codes(params, fam.short_planes, fam.long_planes, cen, d[i]) for i in range(2)]
            out = []
            for order in (0, 1):
                restatement.set_line_order(order)
                out.append(restatement.guided_match_pair(params, cfg, d[0], kp[0], *codes[0], d[1], kp[1], *codes[1], F, band,
                                                         want_ranked=True))
            a, b = out
            assert np.array_equal(a[0], b[0]) and a[1] == b[1] and np.array_equal(a[3], b[3]), seed
            for q in np.flatnonzero(a[3]):
                assert np.array_equal(a[2][q, :a[3][q]], b[2][q, :b[3][q]]), (seed, q)
    finally:
        restatement.set_line_order(0)
    # the two orders do produce different distances (the test is not vacuous) ...
    assert moved_c > 0 and decisions > 4_000_000
    # ... and none of them is close enough to the band edge to change a decision
    assert differing == 0 and near_edge == 0, (differing, near_edge, decisions)
    print(f"f4 line-order bound: {decisions} decisions, {moved_c} distances differ between the orders, "
          f"{near_edge} within 4 ulp of the band edge, {differing} decisions differ")


# ---- the order-independent records checksum (bench.py's and the full-size GPU tests' comparison) ------------
def _mix64(x):
    x = (x + np.uint64(0x9e3779b97f4a7c15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return x ^ (x >> np.uint64(31))


@pytest.mark.parametrize("which", ["restatement", "reference"])
def test_time_match_pairs_checksum_is_the_device_checksum_definition(which, request):
    """chor_time_match_pairs' checksum, from both oracles, equals the formula compact_kernel implements
    (compact_kernels.cuh; tests/test_gpu_parity.py::host_checksum) evaluated over match_pair's own records."""
    import paper_1805_08995_b200 as ch
    orc = request.getfixturevalue(which)
    fam = ch.build_hash_family(FamilyParams())
    d = make_dataset(5, 700, seed=23)
    cen = orc.centering([d[i] for i in range(5)])
    codes = [orc.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, d[i]) for i in range(5)]
    pairs = ch.plan_exhaustive(5, 2, 2)
    cfg = MatchConfig()
    want, total = np.uint64(0), 0
    with np.errstate(over="ignore"):
        for k, (a, b) in enumerate(pairs):
            rec, _ = orc.match_pair(fam.params, cfg, d[a], *codes[a], d[b], *codes[b])
            total += len(rec)
            ka = (np.uint64(k) << np.uint64(32)) | rec["query_index"].astype(np.uint64)
            kb = (rec["train_index"].astype(np.uint64) << np.uint64(32)) | rec["distance_sq"].astype(np.uint64)
            want = want + np.sum(_mix64(_mix64(ka) ^ kb), dtype=np.uint64)
    for threads in (1, 3):
        sec, n, csum = orc.time_match_pairs(fam.params, cfg, [d[i] for i in range(5)], [c[0] for c in codes],
                                            [c[1] for c in codes], pairs, threads)
        assert n == total > 0 and csum == int(want) and sec > 0
