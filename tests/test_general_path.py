"""GPU parity of the general match path (csrc/general_kernels.cuh): what the reference accepts and the tuned kernels
are not laid out for — short codes of 13..32 bits (sparse bucket index), top_k > 32, and match_pair_filtered with a HOST
callback (matcher.hpp:92-105).  Everything goes through the C ABI and is compared bit for bit with the CPU oracle
(the compiled reference where oracle/_ref exists): codes, sorted index, candidate lists, ranked lists, records, statistics.
Nothing here reads /root/reference."""
import numpy as np
import pytest

import oracle_lib
import paper_1805_08995_b200 as ch
from paper_1805_08995_b200.synth import make_dataset

pytestmark = pytest.mark.gpu

BASE = 7000


@pytest.fixture(scope="module")
def oracle():
    return oracle_lib.best()


def install(matcher, family, descs, kps=None):
    for img in list(getattr(matcher, "_test_ids", set())):
        try:
            matcher.evict(img)
        except KeyError:
            pass
    matcher._test_ids = set()
    matcher.set_family(family)
    matcher.set_sub_batch_queries(0)
    matcher.centering_reset()
    for i, d in enumerate(descs):
        matcher.upload(BASE + i, d, None if kps is None else kps[i])
        matcher._test_ids.add(BASE + i)
        matcher.centering_add(BASE + i)
    cen = matcher.centering_apply()
    matcher.hash([BASE + i for i in range(len(descs))])
    return cen


def check_pair(matcher, oracle, fam, cfg, descs, codes, a, b, ranked=True):
    want, wstats, wranked, wcount = oracle.match_pair(fam.params, cfg, descs[a], *codes[a], descs[b], *codes[b], want_ranked=True)
    offs, rec, stats = matcher.match_pairs([(BASE + a, BASE + b)], cfg)
    assert np.array_equal(rec, want), (a, b, len(rec), len(want))
    for key in ("raw_candidates", "verified_queries", "distances", "matches"):
        assert stats[key] == wstats[key], (key, stats[key], wstats[key])
    if ranked:
        got, count = matcher.ranked(BASE + a, BASE + b, cfg)
        assert np.array_equal(count, wcount)
        for q in range(len(count)):
            assert np.array_equal(got[q, : count[q]], wranked[q, : count[q]]), q
    return len(want)


@pytest.mark.parametrize("m,L,n_pts,sigma", [(13, 6, 3000, 8.0), (16, 8, 4000, 8.0), (24, 6, 2500, 4.0), (32, 8, 2500, 1.5)])
def test_sparse_short_codes(matcher, oracle, m, L, n_pts, sigma):
    """short_bits 13..32 (hashing.cpp:30-36): codes, the sorted (code, point) index and the match of pairs, lists of
    pairs included, equal the oracle's."""
    fam = ch.build_hash_family(ch.FamilyParams(short_bits=m, table_count=L))
    descs = list(make_dataset(3, n_pts, seed=100 + m, sigma=sigma))  # (long codes: twins must still share a bucket)
    if m >= 24:
        # buckets of such codes hold one point: repeat half of every image with +-1 noise so that queries see two candidates
        rng = np.random.default_rng(1)
        for i in range(3):
            d, h = descs[i].copy(), n_pts // 2
            d[h: 2 * h] = np.clip(d[:h].astype(np.int16) + rng.integers(-1, 2, size=(h, 128)), 0, 255).astype(np.uint8)
            descs[i] = d
    descs[2] = descs[2][: n_pts // 3]  # ragged
    cen = install(matcher, fam, descs)
    assert np.array_equal(cen, oracle.centering(descs))
    codes = []
    for i, d in enumerate(descs):
        s, l = oracle.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, d)
        c = matcher.codes(BASE + i)
        assert np.array_equal(c.shorts, s) and np.array_equal(c.longs, l), i
        codes.append((s, l))
        sc, sp = matcher.sorted_index(BASE + i)
        for t in range(L):
            order = np.lexsort((np.arange(len(d)), s[:, t]))  # by (code, point): matcher.cpp:34-37
            assert np.array_equal(sp[t], order.astype(np.uint32)) and np.array_equal(sc[t], s[order, t]), (i, t)
    with pytest.raises(ch.UnsupportedError):
        matcher.bucket_index(BASE)  # no dense offsets for these families
    total = 0
    for cfg in (ch.MatchConfig(), ch.MatchConfig(top_k=2, hamming_threshold=55, min_candidates_for_ratio=5),
                ch.MatchConfig(top_k=50, hamming_threshold=128, ratio=0.95)):
        for a, b in ((0, 1), (1, 0), (2, 1), (1, 2)):
            total += check_pair(matcher, oracle, fam, cfg, descs, codes, a, b)
    assert total > 0
    # a pair list in one call: same records, pair by pair
    cfg = ch.MatchConfig()
    pairs = [(0, 1), (1, 2), (2, 0), (1, 0)]
    offs, rec, _ = matcher.match_pairs([(BASE + a, BASE + b) for a, b in pairs], cfg)
    for k, (a, b) in enumerate(pairs):
        want, _ = oracle.match_pair(fam.params, cfg, descs[a], *codes[a], descs[b], *codes[b])
        assert np.array_equal(rec[offs[k]: offs[k + 1]], want), (a, b)


@pytest.mark.parametrize("top_k", [33, 64, 300])
def test_top_k_beyond_the_lane_list(matcher, oracle, top_k):
    """top_k > 32 (validate, matcher.cpp:9-17 asks for >= 2 only) with the default family, empty images included."""
    fam = ch.build_hash_family(ch.FamilyParams())
    descs = list(make_dataset(3, 2500, seed=77))
    descs.append(np.zeros((0, 128), np.uint8))
    cen = install(matcher, fam, descs)
    codes = [oracle.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, d) for d in descs]
    for cfg in (ch.MatchConfig(top_k=top_k), ch.MatchConfig(top_k=top_k, hamming_threshold=64, ratio=0.9),
                ch.MatchConfig(top_k=top_k, hamming_threshold=128, min_candidates_for_ratio=top_k + 7)):
        for a, b in ((0, 1), (2, 0)):
            assert check_pair(matcher, oracle, fam, cfg, descs, codes, a, b) > 0
        for a, b in ((0, 3), (3, 0)):
            assert check_pair(matcher, oracle, fam, cfg, descs, codes, a, b, ranked=False) == 0


def test_top_k_beyond_32_on_large_train_images(matcher, oracle):
    """Train images the tuned path cuts into tiles go through the general kernels whole."""
    fam = ch.build_hash_family(ch.FamilyParams())
    descs = list(make_dataset(2, 14000, seed=5))
    descs[0] = descs[0][:3000]
    cen = install(matcher, fam, descs)
    codes = [oracle.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, d) for d in descs]
    cfg = ch.MatchConfig(top_k=40)
    assert check_pair(matcher, oracle, fam, cfg, descs, codes, 0, 1) > 0


def test_guided_with_top_k_beyond_32(matcher, oracle):
    fam = ch.build_hash_family(ch.FamilyParams())
    rng = np.random.default_rng(9)
    descs = list(make_dataset(2, 2000, seed=12))
    kps = [np.column_stack([rng.uniform(0, 1000, 2000), rng.uniform(0, 800, 2000), np.full(2000, 2.0), np.zeros(2000)]).astype(np.float32)
           for _ in range(2)]
    cen = install(matcher, fam, descs, kps)
    codes = [oracle.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, d) for d in descs]
    F = np.array([[0.0, -1e-3, 0.4], [1e-3, 0.0, -0.5], [-0.4, 0.5, 1.0]])
    cfg = ch.MatchConfig(top_k=48)
    want, _ = oracle.guided_match_pair(fam.params, cfg, descs[0], kps[0], *codes[0], descs[1], kps[1], *codes[1], F, 150.0)[:2]
    offs, rec, _ = matcher.match_pairs_guided([(BASE, BASE + 1)], F.reshape(1, 9), 150.0, cfg)
    assert len(want) > 0 and np.array_equal(rec, want)


def edit(kind, q, cands):
    """Deterministic stand-ins for an arbitrary CandidateFilter (matcher.hpp:92-93): the vector may shrink, be reordered,
    hold duplicates, or come back empty."""
    if kind == "identity":
        return None
    if kind == "reverse":
        return cands[::-1]
    if kind == "thin":
        return [c for c in cands if (c + q) % 3 != 0]
    if kind == "mixed":
        if q % 5 == 0:
            return []
        if q % 5 == 1:
            return cands + cands[:2]      # duplicates stay in the ranking
        if q % 5 == 2:
            return cands[1::2] + cands[0::2]
        return cands
    raise AssertionError(kind)


@pytest.mark.parametrize("m", [8, 14])
@pytest.mark.parametrize("kind", ["identity", "reverse", "thin", "mixed"])
def test_match_pair_filtered_with_a_host_callback(matcher, oracle, m, kind):
    """The candidate lists come from the device, a Python callback edits them, ranking and verification run on the device
    from the edited lists; the oracle side is the reference's own match_pair_filtered driven by the same edits."""
    fam = ch.build_hash_family(ch.FamilyParams(short_bits=m))
    descs = list(make_dataset(2, 2200 if m == 8 else 4000, seed=40 + m))
    cen = install(matcher, fam, descs)
    codes = [oracle.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, d) for d in descs]
    L = fam.params.table_count
    n = len(descs[0])
    offs, cands = matcher.pair_candidates(BASE, BASE + 1)
    lists, lo = [], [0]
    for q in range(n):
        want = oracle.lookup_candidates(m, L, codes[0][0][q], codes[1][0])  # matcher.cpp:53-63
        got = cands[int(offs[q]): int(offs[q + 1])]
        assert np.array_equal(got, want), q
        e = edit(kind, q, want.tolist()) if len(want) else None
        lst = want.tolist() if e is None else e
        lists.extend(lst)
        lo.append(len(lists))
    calls = []

    def cb(q, c):
        calls.append(q)
        return edit(kind, q, c)

    for cfg in (ch.MatchConfig(), ch.MatchConfig(top_k=40, hamming_threshold=60), ch.MatchConfig(top_k=3, min_candidates_for_ratio=6)):
        calls.clear()
        rec, stats = matcher.match_pair_filtered(BASE, BASE + 1, cb, cfg)
        want, wstats = oracle.match_pair_lists(fam.params, cfg, descs[0], *codes[0], descs[1], *codes[1], lo, lists)
        assert np.array_equal(rec, want), (kind, len(rec), len(want))
        assert stats["verified_queries"] == wstats["verified_queries"] and stats["distances"] == wstats["distances"]
        assert calls == [q for q in range(n) if offs[q + 1] > offs[q]]  # called for non-empty lists only, in query order
    if kind == "identity":
        plain, _ = oracle.match_pair(fam.params, ch.MatchConfig(), descs[0], *codes[0], descs[1], *codes[1])
        rec, _ = matcher.match_pair_filtered(BASE, BASE + 1, cb, ch.MatchConfig())
        assert len(plain) > 0 and np.array_equal(rec, plain)


def test_candidate_list_errors(matcher):
    fam = ch.build_hash_family(ch.FamilyParams())
    descs = list(make_dataset(2, 300, seed=3))
    install(matcher, fam, descs)
    offs = np.arange(301, dtype=np.uint64)
    with pytest.raises(ValueError):  # a train point that does not exist
        matcher.match_pair_lists(BASE, BASE + 1, offs, np.full(300, 300, np.uint32))
    with pytest.raises(ValueError):
        matcher.match_pair_lists(BASE, BASE + 1, offs[:-1], np.zeros(299, np.uint32))
    rec, _ = matcher.match_pair_lists(BASE, BASE + 1, np.zeros(301, np.uint64), np.zeros(0, np.uint32))
    assert len(rec) == 0
