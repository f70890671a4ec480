"""Train images larger than the match kernel's shared-memory tile are matched tile by tile (id-range tiles with
their own bucket index, a min pass, a top-k pass and a merge + verification kernel; match_kernels.cuh).  Results,
statistics and ranked lists must be those of the reference's whole-image match_pair (matcher.cpp:141-203)."""
import numpy as np
import pytest

import oracle_lib
import paper_1805_08995_b200 as ch
from paper_1805_08995_b200.synth import make_dataset
from test_gpu_parity import fresh, put, run_pair_case, oracle_codes

pytestmark = pytest.mark.gpu

BASE = 3000


@pytest.fixture(scope="module")
def oracle():
    return oracle_lib.best()


@pytest.fixture(scope="module")
def default_family():
    return ch.build_hash_family(ch.FamilyParams())


CFGS = [ch.MatchConfig(), ch.MatchConfig(top_k=32, hamming_threshold=64, ratio=0.95),
        ch.MatchConfig(top_k=2, min_candidates_for_ratio=5), ch.MatchConfig(hamming_threshold=128, top_k=5),
        ch.MatchConfig(top_k=4, min_candidates_for_ratio=9, hamming_threshold=30)]


@pytest.mark.parametrize("n_i,n_j,shape", [
    (3000, 11000, "uniform"),    # just past the shared-memory capacity: tiles of 8192 + 2808 points
    (12288, 12288, "uniform"),
    (500, 24577, "sift"),        # 3 full tiles + one of a single point; skewed buckets inside the tiles
    (20000, 9000, "uniform"),    # large query image, train image below the capacity: the ordinary path
    (1200, 65536, "uniform"),    # the envelope's edge: the largest image the device path holds (u16 point ids), 8 tiles
    (65536, 3000, "uniform"),    # ... and as the query image
])
def test_tiled_match_bit_exact(matcher, oracle, default_family, n_i, n_j, shape):
    fresh(matcher, default_family)
    d = make_dataset(2, max(n_i, n_j), seed=71 + n_j, shape=shape)
    want = run_pair_case(matcher, oracle, default_family, d[0][:n_i], d[1][:n_j], CFGS, ids=(BASE, BASE + 1))
    if shape == "uniform":
        assert len(want) > 0.1 * min(n_i, n_j)


def test_candidates_tie_across_tiles(matcher, oracle, default_family):
    """The same descriptors in several tiles: equal Hamming keys up to the id, equal Euclidean distances; rank
    order and the tie rules (earlier rank wins, zero second distance rejects) must survive the merge."""
    fresh(matcher, default_family)
    d = make_dataset(2, 6000, seed=5)
    train = np.concatenate([d[1], d[1][::-1], d[1][:3000]])     # 15,000 points, every row 2-3 times
    run_pair_case(matcher, oracle, default_family, d[0], train, [ch.MatchConfig(), ch.MatchConfig(top_k=3)],
                  ids=(BASE, BASE + 1))
    near = train.copy()
    near[6000:, 0] ^= 1                                          # near-duplicates: tiny nonzero second distance
    run_pair_case(matcher, oracle, default_family, d[0], near, [ch.MatchConfig(ratio=0.99)], ids=(BASE, BASE + 1))


@pytest.mark.parametrize("params,n", [(ch.FamilyParams(10, 96, 4, 99), 15000), (ch.FamilyParams(6, 64, 8, 2), 14000),
                                      (ch.FamilyParams(3, 32, 3, 8), 12000)])
def test_tiled_other_families(matcher, oracle, params, n):
    fam = ch.build_hash_family(params)
    fresh(matcher, fam)
    d = make_dataset(2, n, seed=13)
    tau = min(40, params.long_bits)
    run_pair_case(matcher, oracle, fam, d[0][:1500], d[1], [ch.MatchConfig(hamming_threshold=tau // 2),
                                                           ch.MatchConfig(hamming_threshold=params.long_bits, top_k=7)],
                  ids=(BASE, BASE + 1))


def test_mixed_pair_list_keeps_pair_order(matcher, oracle, default_family):
    """Small and large train images interleaved: sub-batches are cut where the kind changes, results stay in
    pair order; replacing / evicting a large image recycles its tile slots."""
    fresh(matcher, default_family)
    sizes = [2000, 12000, 3000, 17000, 2500]
    d = [make_dataset(1, n, seed=100 + n)[0] for n in sizes]
    cen = oracle.centering(d)
    matcher.set_centering(cen)
    ids = [BASE + i for i in range(len(sizes))]
    for i, x in zip(ids, d):
        put(matcher, i, x)
    matcher.hash(ids)
    codes = [oracle_codes(oracle, default_family, cen, x) for x in d]
    pairs = [(0, 1), (0, 2), (1, 3), (3, 1), (2, 4), (4, 3), (1, 0), (3, 3)]
    cfg = ch.MatchConfig()
    offs, rec, stats = matcher.match_pairs([(BASE + a, BASE + b) for a, b in pairs], cfg)
    assert stats["pairs"] == len(pairs)
    raw = 0
    for k, (a, b) in enumerate(pairs):
        want, ws = oracle.match_pair(default_family.params, cfg, d[a], *codes[a], d[b], *codes[b])
        assert np.array_equal(rec[offs[k]:offs[k + 1]], want), (a, b)
        raw += ws["raw_candidates"]
    assert stats["raw_candidates"] == raw
    st = matcher.match_pairs_device([(BASE + a, BASE + b) for a, b in pairs], cfg)
    assert st["matches"] == len(rec)
    # replace a large image by a small one and a small one by a large one, evict another: slots are recycled
    d[1], d[0] = d[1][:1000], make_dataset(1, 13000, seed=7)[0]
    put(matcher, ids[1], d[1])
    put(matcher, ids[0], d[0])
    matcher.evict(ids[3])
    matcher._test_ids.discard(ids[3])
    matcher.hash([ids[0], ids[1]])
    codes[0] = oracle_codes(oracle, default_family, cen, d[0])
    codes[1] = oracle_codes(oracle, default_family, cen, d[1])
    for a, b in ((1, 0), (2, 0), (0, 1)):
        want, _ = oracle.match_pair(default_family.params, cfg, d[a], *codes[a], d[b], *codes[b])
        _, got, _ = matcher.match_pairs([(BASE + a, BASE + b)], cfg)
        assert np.array_equal(got, want), (a, b)


def test_external_codes_build_the_tiles(matcher, oracle, default_family):
    """chgpu_upload_codes (the code-cache resume path) builds the tile indices as well."""
    fresh(matcher, default_family)
    d = make_dataset(2, 12500, seed=3)
    cen = oracle.centering(list(d))
    matcher.set_centering(cen)
    cfg = ch.MatchConfig()
    codes = [oracle_codes(oracle, default_family, cen, x) for x in d]
    for i in range(2):
        put(matcher, BASE + i, d[i])
        matcher.upload_codes(BASE + i, ch.ImageCodes(default_family.params, codes[i][0], codes[i][1]))
    want, _ = oracle.match_pair(default_family.params, cfg, d[0], *codes[0], d[1], *codes[1])
    _, got, _ = matcher.match_pairs([(BASE, BASE + 1)], cfg)
    assert np.array_equal(got, want)


def test_slot_churn_with_tiles(matcher, oracle, default_family):
    """Uploads, replacements and evictions of small and large images in random order: image slots, hidden tile
    slots and arena blocks are recycled; what is resident at the end still matches like the reference."""
    fresh(matcher, default_family)
    rng = np.random.default_rng(12)
    pool = {n: make_dataset(1, n, seed=300 + n)[0] for n in (500, 3000, 11500, 13000, 17000)}
    cen = oracle.centering(list(pool.values()))
    matcher.set_centering(cen)
    resident = {}
    for step in range(60):
        slot = BASE + int(rng.integers(0, 6))
        if slot in resident and rng.random() < 0.3:
            matcher.evict(slot)
            matcher._test_ids.discard(slot)
            del resident[slot]
        else:
            n = int(rng.choice(list(pool)))
            put(matcher, slot, pool[n])
            resident[slot] = n
    ids = sorted(resident)
    assert len(ids) >= 2
    matcher.hash(ids)
    cfg = ch.MatchConfig()
    codes = {n: oracle_codes(oracle, default_family, cen, pool[n]) for n in set(resident.values())}
    pairs = [(a, b) for a in ids for b in ids if a != b][:8]
    offs, rec, _ = matcher.match_pairs(pairs, cfg)
    for k, (a, b) in enumerate(pairs):
        na, nb = resident[a], resident[b]
        want, _ = oracle.match_pair(default_family.params, cfg, pool[na], *codes[na], pool[nb], *codes[nb])
        assert np.array_equal(rec[offs[k]:offs[k + 1]], want), (na, nb)
