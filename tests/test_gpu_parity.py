"""GPU parity suite (run with `-m gpu` on a B200).  Every check goes through the C ABI
(libchgpu.so) and compares with the CPU oracle on the same inputs:
  - hash codes, bucket CSR and ranked candidate lists: bit-exact;
  - match records: bit-exact (stronger than the 99.9 % agreement north_star allows);
  - golden vectors produced by the compiled reference (tests/golden);
  - size-independent properties at BASELINE.json's config-2 size.
Nothing here reads /root/reference."""
import struct

import numpy as np
import pytest

import oracle_lib
import paper_1805_08995_b200 as ch
from paper_1805_08995_b200.synth import make_dataset
from test_oracle import GOLDEN_CFGS

pytestmark = pytest.mark.gpu

BASE = 1000  # image ids used by this module


def fresh(matcher, family):
    """Drops every image this module may have left and installs `family`."""
    for img in list(getattr(matcher, "_test_ids", set())):
        try:
            matcher.evict(img)
        except KeyError:
            pass
    matcher._test_ids = set()
    matcher.set_family(family)
    matcher.set_sub_batch_queries(0)


@pytest.fixture(autouse=True, params=["join_by_size", "join_always"])
def join_mode(request, matcher):
    """Every test of this module runs twice: with the tensor-core Hamming pass (join_kernels.cuh) taken by the library's
    own rule (sub-batches of >= 20 points per bucket: none of the small cases here) and forced for every sub-batch it can
    serve, so that the pass and the active-list form of the match kernel see every edge case the plain kernel sees."""
    matcher.set_join(True, 0 if request.param == "join_always" else 20)
    yield request.param
    matcher.set_join(True, 20)


def put(matcher, image_id, desc, kp=None):
    matcher.upload(image_id, desc, kp)
    matcher._test_ids.add(image_id)


@pytest.fixture(scope="module")
def oracle():
    return oracle_lib.best()  # the compiled reference where it exists, else the pinned restatement


@pytest.fixture(scope="module")
def default_family():
    return ch.build_hash_family(ch.FamilyParams())


def oracle_codes(oracle, fam, cen, desc, rr=3):
    return oracle.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, desc, rr)


def mix64(x):
    x = (x + np.uint64(0x9e3779b97f4a7c15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return x ^ (x >> np.uint64(31))


def host_checksum(offsets, records):
    """Same order-independent checksum compact_kernel accumulates on the device."""
    with np.errstate(over="ignore"):
        pair = np.repeat(np.arange(len(offsets) - 1, dtype=np.uint64), np.diff(offsets).astype(np.int64))
        a = (pair << np.uint64(32)) | records["query_index"].astype(np.uint64)
        b = (records["train_index"].astype(np.uint64) << np.uint64(32)) | records["distance_sq"].astype(np.uint64)
        return int(np.sum(mix64(mix64(a) ^ b), dtype=np.uint64))


# ---- golden vectors -------------------------------------------------------------------------------
def test_codes_buckets_matches_equal_golden(matcher, golden, default_family):
    g = golden["small_dataset"]
    fresh(matcher, default_family)
    desc = g["desc"]
    for i in range(3):
        put(matcher, BASE + i, desc[i])
    # centering: exact integer sums on the device, one division on the host
    matcher.centering_reset()
    for i in range(3):
        matcher.centering_add(BASE + i)
    sums, count = matcher.centering_sums()
    assert count == 900 and np.array_equal(sums, desc.reshape(-1, 128).astype(np.uint64).sum(0))
    cen = matcher.centering_apply()
    assert np.array_equal(cen, g["centering"])

    import hashlib
    for rr in (0, 7, 3):
        matcher.hash([BASE, BASE + 1, BASE + 2], rr)
        for i in range(3):
            c = matcher.codes(BASE + i)
            if rr == 3:
                assert np.array_equal(c.shorts, g[f"shorts{i}"]) and np.array_equal(c.longs, g[f"longs{i}"])
            else:
                assert hashlib.sha256(c.shorts.tobytes()).hexdigest() == str(g[f"shorts{i}_rr{rr}_sha"])
                assert hashlib.sha256(c.longs.tobytes()).hexdigest() == str(g[f"longs{i}_rr{rr}_sha"])
    bi = matcher.bucket_index(BASE + 1)
    assert np.array_equal(bi.offsets, g["offs1"]) and np.array_equal(bi.points, g["pts1"])

    for tag, cfg in GOLDEN_CFGS.items():
        pairs = [(BASE + a, BASE + b) for a, b in ((0, 1), (1, 2), (2, 0))]
        offs, rec, stats = matcher.match_pairs(pairs, cfg)
        for k, (a, b) in enumerate(((0, 1), (1, 2), (2, 0))):
            assert np.array_equal(rec[offs[k]:offs[k + 1]], g[f"rec_{tag}_{a}{b}"]), (tag, a, b)
            ranked, rc = matcher.ranked(BASE + a, BASE + b, cfg)
            assert np.array_equal(rc, g[f"rcount_{tag}_{a}{b}"]), (tag, a, b)
            gr = g[f"ranked_{tag}_{a}{b}"]
            for q in range(len(rc)):
                assert np.array_equal(ranked[q, :rc[q]], gr[q, :rc[q]]), (tag, a, b, q)
        gs = [g[f"stats_{tag}_{a}{b}"] for a, b in ((0, 1), (1, 2), (2, 0))]
        assert stats["raw_candidates"] == sum(int(s[0]) for s in gs)
        assert stats["verified_queries"] == sum(int(s[4]) for s in gs)
        assert stats["distances"] == sum(int(s[5]) for s in gs)
        assert stats["matches"] == sum(int(s[6]) for s in gs) == len(rec)


# ---- hash build vs oracle ---------------------------------------------------------------------------
@pytest.mark.parametrize("params,n,shape", [
    (ch.FamilyParams(), 1000, "uniform"),            # BASELINE config 1 size
    (ch.FamilyParams(), 4096, "sift"),
    (ch.FamilyParams(10, 96, 4, 99), 777, "uniform"),
    (ch.FamilyParams(12, 128, 8, 3), 513, "sift"),
    (ch.FamilyParams(1, 2, 1, 1), 65, "uniform"),     # smallest legal family
    (ch.FamilyParams(5, 33, 7, 4), 64, "uniform"),    # code words straddle 32-bit boundaries
])
def test_codes_and_buckets_bit_exact(matcher, oracle, params, n, shape):
    fam = ch.build_hash_family(params)
    fresh(matcher, fam)
    desc = make_dataset(2, n, seed=21, shape=shape)
    cen = oracle.centering(list(desc))
    matcher.set_centering(cen)
    put(matcher, BASE, desc[0])
    put(matcher, BASE + 1, desc[1])
    for rr in (3, 0, 1, 2, 4, 5, 6, 7):
        matcher.hash([BASE, BASE + 1], rr)
        for i in range(2):
            s, l = oracle_codes(oracle, fam, cen, desc[i], rr)
            c = matcher.codes(BASE + i)
            assert np.array_equal(c.shorts, s), (rr, i)
            assert np.array_equal(c.longs, l), (rr, i)
    s, _ = oracle_codes(oracle, fam, cen, desc[1])
    offs, pts = oracle.build_bucket_index(params.short_bits, params.table_count, s)
    bi = matcher.bucket_index(BASE + 1)
    assert np.array_equal(bi.offsets, offs) and np.array_equal(bi.points, pts)


def test_near_tie_projections_keep_their_sign(matcher, oracle, default_family):
    """Descriptors equal to the centering give dot == 0 exactly -> bit 0; and a large
    random sample has the same bits as the oracle even for |dot| < 1 (the fp64 exact-order claim)."""
    fresh(matcher, default_family)
    cen = np.full(128, 77.0)
    matcher.set_centering(cen)
    put(matcher, BASE, np.full((3, 128), 77, np.uint8))
    matcher.hash([BASE])
    c = matcher.codes(BASE)
    assert not c.shorts.any() and not c.longs.any()
    desc = make_dataset(1, 8192, seed=5)[0]
    cen = oracle.centering([desc])
    matcher.set_centering(cen)
    put(matcher, BASE + 1, desc)
    matcher.hash([BASE + 1])
    s, l = oracle_codes(oracle, default_family, cen, desc)
    c = matcher.codes(BASE + 1)
    assert np.array_equal(c.shorts, s) and np.array_equal(c.longs, l)
    dots = (desc.astype(np.float64) - cen) @ default_family.long_planes.T
    assert (np.abs(dots) < 1.0).sum() > 100, "sample must contain near-zero projections"


def test_batch_upload_equals_single_uploads(matcher, default_family):
    fresh(matcher, default_family)
    d = make_dataset(5, 700, seed=77)
    kp = np.random.default_rng(1).uniform(0, 100, (5, 700, 4)).astype(np.float32)
    ids = [BASE + i for i in range(5)]
    pinned = matcher.pinned_empty(d.shape, np.uint8)
    pinned[:] = d
    for src, k in ((pinned, None), (np.ascontiguousarray(d), kp)):   # pinned / pageable source
        matcher.upload_many(ids, src, k)
        matcher._test_ids.update(ids)
        for i in range(5):
            got_d, got_k = matcher.descriptors(ids[i])
            assert np.array_equal(got_d, d[i])
            assert np.array_equal(got_k, kp[i] if k is not None else np.zeros((700, 4), np.float32))
    matcher.upload_many([], np.zeros((0, 700, 128), np.uint8))


def test_batched_centering_sums_equal_the_per_image_sums(matcher, oracle, default_family):
    fresh(matcher, default_family)
    sizes = [0, 1, 31, 1000, 4097, 20000]
    d = [make_dataset(1, max(n, 1), seed=200 + n)[0][:n] for n in sizes]
    for i, x in enumerate(d):
        put(matcher, BASE + i, x)
    ids = [BASE + i for i in range(len(d))]
    matcher.centering_reset()
    for i in ids:
        matcher.centering_add(i)
    one, cnt1 = matcher.centering_sums()
    matcher.centering_reset()
    matcher.centering_add_many(ids)
    many, cnt2 = matcher.centering_sums()
    assert cnt1 == cnt2 == sum(sizes) and np.array_equal(one, many)
    assert np.array_equal(one, np.concatenate(d).astype(np.uint64).sum(axis=0))
    assert np.array_equal(matcher.centering_apply(), oracle.centering([x for x in d if len(x)]))


# ---- match vs oracle --------------------------------------------------------------------------------
def run_pair_case(matcher, oracle, fam, desc_i, desc_j, cfgs, ids=(BASE, BASE + 1)):
    cen = oracle.centering([desc_i, desc_j]) if len(desc_i) + len(desc_j) else np.zeros(128)
    matcher.set_centering(cen)
    put(matcher, ids[0], desc_i)
    put(matcher, ids[1], desc_j)
    matcher.hash(list(ids))
    ci = oracle_codes(oracle, fam, cen, desc_i)
    cj = oracle_codes(oracle, fam, cen, desc_j)
    for cfg in cfgs:
        want, wstats, wranked, wrc = oracle.match_pair(fam.params, cfg, desc_i, *ci, desc_j, *cj, want_ranked=True)
        offs, rec, stats = matcher.match_pairs([ids], cfg)
        assert offs.tolist() == [0, len(want)]
        assert np.array_equal(rec, want), cfg
        assert stats["raw_candidates"] == wstats["raw_candidates"]
        assert stats["verified_queries"] == wstats["verified_queries"]
        assert stats["distances"] == wstats["distances"]
        ranked, rc = matcher.ranked(ids[0], ids[1], cfg)
        assert np.array_equal(rc, wrc[: len(rc)])
        for q in np.nonzero(rc)[0]:
            assert np.array_equal(ranked[q, :rc[q]], wranked[q, :rc[q]]), (cfg, q)
    return want


CFGS = [ch.MatchConfig(), ch.MatchConfig(hamming_threshold=128), ch.MatchConfig(top_k=2, min_candidates_for_ratio=5),
        ch.MatchConfig(top_k=32, hamming_threshold=64, ratio=0.95), ch.MatchConfig(top_k=3, hamming_threshold=50, ratio=0.5,
                                                                                     min_candidates_for_ratio=0)]


@pytest.mark.parametrize("n_i,n_j,shape", [
    (1000, 1000, "uniform"),   # BASELINE config 1
    (4096, 4096, "uniform"),   # config 2 image size
    (4096, 3000, "sift"),
    (8192, 8192, "uniform"),   # config 3 image size: train codes fill 128 KiB of shared memory
    (8192, 8192, "sift"),      # skewed buckets
    (777, 13000, "uniform"),   # ragged, near the shared-memory capacity
])
def test_match_bit_exact(matcher, oracle, default_family, n_i, n_j, shape):
    fresh(matcher, default_family)
    n = max(n_i, n_j)
    d = make_dataset(2, n, seed=31 + n_i, shape=shape)
    want = run_pair_case(matcher, oracle, default_family, d[0][:n_i], d[1][:n_j], CFGS)
    if shape == "uniform":
        assert len(want) > 0.2 * min(n_i, n_j), "twins must match"


@pytest.mark.parametrize("n,shape", [(16384, "uniform"), (32768, "uniform"), (20000, "sift")])
def test_match_large_images_global_gather_and_multipass(matcher, oracle, default_family, n, shape):
    """Config-5 sizes: train codes no longer fit shared memory (global-gather variant) and the raw
    candidate count per query exceeds one ranking pass (merge path)."""
    fresh(matcher, default_family)
    d = make_dataset(2, n, seed=41, shape=shape)
    run_pair_case(matcher, oracle, default_family, d[0], d[1], [ch.MatchConfig(), ch.MatchConfig(top_k=4, hamming_threshold=45)])


@pytest.mark.parametrize("params", [ch.FamilyParams(10, 96, 4, 99), ch.FamilyParams(6, 64, 8, 2),
                                    ch.FamilyParams(12, 128, 2, 3), ch.FamilyParams(3, 32, 3, 8)])
def test_match_other_families(matcher, oracle, params):
    fam = ch.build_hash_family(params)
    fresh(matcher, fam)
    d = make_dataset(2, 2000, seed=51)
    tau = min(40, params.long_bits)
    run_pair_case(matcher, oracle, fam, d[0], d[1], [ch.MatchConfig(hamming_threshold=tau // 2),
                                                     ch.MatchConfig(hamming_threshold=params.long_bits, top_k=7)])


def test_edge_cases(matcher, oracle, default_family):
    fresh(matcher, default_family)
    d = make_dataset(2, 300, seed=61)
    empty = np.zeros((0, 128), np.uint8)
    cfg = [ch.MatchConfig()]
    assert len(run_pair_case(matcher, oracle, default_family, d[0], empty, cfg)) == 0      # fsJ empty
    assert len(run_pair_case(matcher, oracle, default_family, empty, d[1], cfg)) == 0
    assert len(run_pair_case(matcher, oracle, default_family, d[0], d[1][:1], cfg)) == 0   # ratio undecidable
    # exact duplicates: second distance 0 -> rejection; duplicated + distinct rows mixed
    dup = np.repeat(d[0][:40], 3, axis=0)
    run_pair_case(matcher, oracle, default_family, d[0][:40], dup, cfg)
    run_pair_case(matcher, oracle, default_family, dup, dup, cfg)
    # image matched against itself (every query has a zero-distance twin)
    run_pair_case(matcher, oracle, default_family, d[0], d[0], cfg)
    # sizes around warp / tile boundaries
    for n_i, n_j in ((1, 300), (31, 33), (32, 64), (33, 65), (255, 257)):
        run_pair_case(matcher, oracle, default_family, d[0][:n_i], d[1][:n_j], cfg)


def test_errors_follow_the_reference(matcher, default_family):
    fresh(matcher, default_family)
    d = make_dataset(1, 64, seed=1)[0]
    put(matcher, BASE, d)
    put(matcher, BASE + 1, d)
    with pytest.raises(ch.LogicError):          # codes not computed
        matcher.match_pairs([(BASE, BASE + 1)], ch.MatchConfig())
    m2 = ch.Matcher(0)
    try:
        m2.set_family(default_family)
        m2.upload(1, d)
        with pytest.raises(ch.LogicError):      # hashing.cpp:131-132 centering not set
            m2.hash([1])
        with pytest.raises(ValueError):         # hashing.hpp:28-29
            m2.set_centering(np.zeros(128))
            m2.hash([1], 8)
        with pytest.raises(ValueError):         # hashing.cpp:60 empty stream
            m2.centering_reset()
            m2.centering_apply()
    finally:
        m2.close()
    matcher.set_centering(np.full(128, 127.5))
    matcher.hash([BASE, BASE + 1])
    for bad in (ch.MatchConfig(top_k=1), ch.MatchConfig(hamming_threshold=129), ch.MatchConfig(ratio=1.0),
                ch.MatchConfig(ratio=0.0), ch.MatchConfig(reduce_rounds=8), ch.MatchConfig(reduce_rounds=-1)):
        with pytest.raises(ValueError):         # matcher.cpp:9-17
            matcher.match_pairs([(BASE, BASE + 1)], bad)
    matcher.match_pairs([(BASE, BASE + 1)], ch.MatchConfig(top_k=33))  # general path (tests/test_general_path.py)
    with pytest.raises(KeyError):
        matcher.match_pairs([(BASE, 999999)], ch.MatchConfig())
    with pytest.raises(ch.UnsupportedError):
        matcher.upload(BASE + 2, np.zeros((65537, 128), np.uint8))
    m3 = ch.Matcher(0)
    try:
        m3.set_family(ch.build_hash_family(ch.FamilyParams(short_bits=13)))  # sparse bucket index: general path
        with pytest.raises(ch.UnsupportedError):
            m3.set_family(ch.build_hash_family(ch.FamilyParams(table_count=9)))
    finally:
        m3.close()


# ---- descriptor load -------------------------------------------------------------------------------
def chft_blob(desc, kp, version=1, magic=b"CHFT"):
    n = len(desc)
    out = bytearray(magic + struct.pack("<III", version, n, 0))
    for i in range(n):
        out += kp[i].astype("<f4").tobytes() + desc[i].tobytes()
    return bytes(out)


def test_chft_load_and_faults(matcher, oracle, default_family):
    fresh(matcher, default_family)
    d = make_dataset(1, 1234, seed=71)[0]
    kp = np.random.default_rng(0).normal(size=(1234, 4)).astype(np.float32)
    blob = chft_blob(d, kp)
    assert len(blob) == 16 + 1234 * 144                     # feature_io.hpp:88-89
    assert matcher.upload_chft(BASE, blob) == 1234
    matcher._test_ids.add(BASE)
    got_d, got_kp = matcher.descriptors(BASE)
    assert np.array_equal(got_d, d) and np.array_equal(got_kp, kp)
    # trailing bytes are ignored like the stream reader does; empty files are valid
    assert matcher.upload_chft(BASE, blob + b"xx") == 1234
    assert matcher.upload_chft(BASE + 1, chft_blob(d[:0], kp[:0])) == 0
    matcher._test_ids.add(BASE + 1)
    assert matcher.points(BASE + 1) == 0
    # the loaded image hashes and matches like an uploaded one
    put(matcher, BASE + 2, d)
    cen = oracle.centering([d])
    matcher.set_centering(cen)
    matcher.hash([BASE, BASE + 2])
    a, b = matcher.codes(BASE), matcher.codes(BASE + 2)
    assert np.array_equal(a.shorts, b.shorts) and np.array_equal(a.longs, b.longs)
    # fault classes and byte offsets of parse_features_blob (engine.cpp:458-472)
    for bad, fault, off in ((blob[:10], "Truncated", 10), (b"XHFT" + blob[4:], "BadMagic", 0),
                            (chft_blob(d, kp, version=2), "BadVersion", 4), (blob[:5000], "Truncated", 5000)):
        with pytest.raises(ch.FeatureFileError) as ei:
            matcher.upload_chft(BASE + 3, bad)
        assert ei.value.fault == fault and ei.value.byte_offset == off


def test_external_codes_round_trip(matcher, oracle, default_family):
    """Codes computed elsewhere (a CHCC cache, the CPU reference) can be installed and matched."""
    fresh(matcher, default_family)
    d = make_dataset(2, 1500, seed=81)
    cen = oracle.centering(list(d))
    ci = oracle_codes(oracle, default_family, cen, d[0])
    cj = oracle_codes(oracle, default_family, cen, d[1])
    put(matcher, BASE, d[0])
    put(matcher, BASE + 1, d[1])
    matcher.upload_codes(BASE, ch.ImageCodes(default_family.params, *ci))
    matcher.upload_codes(BASE + 1, ch.ImageCodes(default_family.params, *cj))
    want, _ = oracle.match_pair(default_family.params, ch.MatchConfig(), d[0], *ci, d[1], *cj)
    _, rec, _ = matcher.match_pairs([(BASE, BASE + 1)], ch.MatchConfig())
    assert np.array_equal(rec, want)
    with pytest.raises(ValueError):
        bad = ci[0].copy()
        bad[0, 0] = 256
        matcher.upload_codes(BASE, ch.ImageCodes(default_family.params, bad, ci[1]))


# ---- pair lists, batching, sinks ---------------------------------------------------------------------
def test_pair_list_batching_is_invariant(matcher, oracle, default_family):
    """SPEC criterion 8 (worker invariance): results do not depend on how the pair list is cut
    into sub-batches, shards or work units; sink delivery is in pair order."""
    fresh(matcher, default_family)
    k, n = 12, 1000
    d = make_dataset(k, n, seed=91)
    cen = oracle.centering(list(d))
    matcher.set_centering(cen)
    for i in range(k):
        put(matcher, BASE + i, d[i])
    matcher.hash([BASE + i for i in range(k)])
    pairs = ch.plan_exhaustive(k, 3, 2) + BASE
    cfg = ch.MatchConfig()
    offs, rec, stats = matcher.match_pairs(pairs, cfg)
    assert stats["pairs"] == 66 and stats["match_launches"] == 1
    # oracle on a few pairs of the list
    codes = [oracle_codes(oracle, default_family, cen, d[i]) for i in range(k)]
    for idx in (0, 17, 65):
        a, b = int(pairs[idx, 0]) - BASE, int(pairs[idx, 1]) - BASE
        want, _ = oracle.match_pair(default_family.params, cfg, d[a], *codes[a], d[b], *codes[b])
        assert np.array_equal(rec[offs[idx]:offs[idx + 1]], want)
    # many small sub-batches, delivered through the sink
    matcher.set_sub_batch_queries(5 * n)
    chunks = []
    st2 = matcher.match_pairs_stream(pairs, cfg, lambda first, o, r: chunks.append((first, o.copy(), r.copy())))
    assert st2["match_launches"] == 14 and [c[0] for c in chunks] == list(range(0, 66, 5))
    cat = np.concatenate([c[2] for c in chunks])
    assert np.array_equal(cat, rec)
    for first, o, r in chunks:
        assert np.array_equal(o + offs[first], offs[first:first + len(o)])
    offs3, rec3, st3 = matcher.match_pairs(pairs, cfg)
    assert np.array_equal(offs3, offs) and np.array_equal(rec3, rec) and st3["match_launches"] == 14
    matcher.set_sub_batch_queries(0)
    # shards of the list (the multi-GPU split) concatenate to the whole
    parts = []
    for r in range(3):
        a, b = ch.shard_range(len(pairs), r, 3)
        parts.append(matcher.match_pairs(pairs[a:b], cfg)[1])
    assert np.array_equal(np.concatenate(parts), rec)
    # device-resident run reports the same counters and checksum
    st4 = matcher.match_pairs_device(pairs, cfg)
    assert st4["matches"] == len(rec) and st4["records_checksum"] == host_checksum(offs, rec)
    assert st4["raw_candidates"] == stats["raw_candidates"] and st4["distances"] == stats["distances"]
    # capacity too small -> ENOMEM with the required size, offsets still complete
    with pytest.raises(MemoryError):
        matcher.match_pairs(pairs, cfg, capacity=10)


def test_sub_batches_rounded_to_the_sm_count(matcher, default_family, monkeypatch):
    """A sub-batch holds a multiple of the SM count of pairs (one unit per pair in the persistent grid); where the cut
    falls never changes a record."""
    fresh(matcher, default_family)
    k, n = 36, 256
    d = make_dataset(k, n, seed=93)
    matcher.centering_reset()
    for i in range(k):
        put(matcher, BASE + i, d[i])
        matcher.centering_add(BASE + i)
    matcher.centering_apply()
    matcher.hash([BASE + i for i in range(k)])
    pairs = ch.plan_exhaustive(k, 4, 3) + BASE  # 630 pairs
    cfg = ch.MatchConfig()
    sms = matcher.device_props()["sm_count"]
    offs, rec, st = matcher.match_pairs(pairs, cfg)
    assert st["match_launches"] == 1
    try:
        matcher.set_sub_batch_queries((4 * sms + 5) * n)  # room for 4 * sms + 5 pairs: the cut moves down to 4 * sms
        chunks = []
        st2 = matcher.match_pairs_stream(pairs, cfg, lambda first, o, r: chunks.append((first, len(o) - 1, r.copy())))
        want_first = list(range(0, len(pairs), 4 * sms))
        assert [c[0] for c in chunks] == want_first and chunks[0][1] == min(4 * sms, len(pairs))
        assert np.array_equal(np.concatenate([c[2] for c in chunks]), rec)
        monkeypatch.setenv("CHGPU_NO_SUBBATCH_ROUNDING", "1")
        chunks2 = []
        matcher.match_pairs_stream(pairs, cfg, lambda first, o, r: chunks2.append((first, len(o) - 1, r.copy())))
        assert [c[0] for c in chunks2] == list(range(0, len(pairs), 4 * sms + 5))
        assert np.array_equal(np.concatenate([c[2] for c in chunks2]), rec)
    finally:
        matcher.set_sub_batch_queries(0)


def test_config2_properties_full_size(matcher, default_family):
    """BASELINE config 2 (100 images x 4,096 descriptors, 4,950 pairs) through the pair-list path;
    checked with properties that need no oracle run."""
    fresh(matcher, default_family)
    k, n = 100, 4096
    d = make_dataset(k, n, seed=7)
    for i in range(k):
        put(matcher, BASE + i, d[i])
    matcher.centering_reset()
    for i in range(k):
        matcher.centering_add(BASE + i)
    cen = matcher.centering_apply()
    assert np.array_equal(cen, d.reshape(-1, 128).astype(np.uint64).sum(0).astype(np.float64) / (k * n))
    matcher.hash([BASE + i for i in range(k)])
    pairs = ch.plan_exhaustive(k, 10, 4) + BASE
    cfg = ch.MatchConfig()
    offs, rec, stats = matcher.match_pairs(pairs, cfg)
    assert stats["pairs"] == 4950 and len(offs) == 4951 and offs[-1] == len(rec) == stats["matches"]
    # ascending query index inside every pair, at most one record per query (matcher.hpp:96-97)
    seg = np.repeat(np.arange(4950), np.diff(offs).astype(np.int64))
    same = seg[1:] == seg[:-1]
    assert (np.diff(rec["query_index"].astype(np.int64))[same] > 0).all()
    assert rec["query_index"].max() < n and rec["train_index"].max() < n
    # every record's distance is the exact squared distance of the two descriptors it names
    pick = np.random.default_rng(0).choice(len(rec), 20000, replace=False)
    pa, pb = pairs[seg[pick], 0] - BASE, pairs[seg[pick], 1] - BASE
    qa = d[pa, rec["query_index"][pick]].astype(np.int64)
    tb = d[pb, rec["train_index"][pick]].astype(np.int64)
    assert np.array_equal(((qa - tb) ** 2).sum(1).astype(np.float64), rec["distance_sq"][pick])
    # twins (slot s in both images) dominate: recall of the planted correspondences
    twins = int(np.ceil(0.3 * n))
    planted = rec["query_index"] == rec["train_index"]
    assert (rec["query_index"][planted] < twins).all()
    assert planted.sum() / (4950 * twins) > 0.90 and planted.mean() > 0.99
    # checksum of checksums: device-only path and host delivery agree
    st2 = matcher.match_pairs_device(pairs, cfg)
    assert st2["records_checksum"] == host_checksum(offs, rec) and st2["matches"] == len(rec)
    # swapping query and train image is a different computation with a consistent answer
    a, b = int(pairs[0, 0]), int(pairs[0, 1])
    _, r_ab, _ = matcher.match_pairs([(a, b)], cfg)
    _, r_ba, _ = matcher.match_pairs([(b, a)], cfg)
    ab = set(zip(r_ab["query_index"].tolist(), r_ab["train_index"].tolist()))
    ba = set(zip(r_ba["train_index"].tolist(), r_ba["query_index"].tolist()))
    assert len(ab & ba) > 0.9 * min(len(ab), len(ba))


def test_config2_full_size_records_equal_the_oracle(matcher, oracle, default_family):
    """BASELINE config 2 at full size against the ORACLE: all 4,950 pairs of 100 x 4,096 descriptors are matched by the CPU
    reference (all host threads) and every record is compared through the order-independent checksum the compaction
    kernel accumulates on the device — pair position, query, train index and distance of all ~6 M records."""
    import os
    fresh(matcher, default_family)
    k, n = 100, 4096
    d = make_dataset(k, n, seed=7)
    ids = np.arange(BASE, BASE + k, dtype=np.uint32)
    matcher.upload_many(ids, np.ascontiguousarray(d))
    matcher._test_ids.update(int(i) for i in ids)
    matcher.centering_reset()
    matcher.centering_add_many(ids)
    cen = matcher.centering_apply()
    matcher.hash(ids)
    codes = [matcher.codes(int(i)) for i in ids]
    p = default_family.params
    for i in (0, 37, 99):  # the device codes the oracle run is fed are the oracle's own (bit-exact hash build)
        s, l = oracle.compute_codes(p, default_family.short_planes, default_family.long_planes, cen, d[i])
        assert np.array_equal(codes[i].shorts, s) and np.array_equal(codes[i].longs, l)
    pairs = ch.plan_exhaustive(k, 10, 4)
    cfg = ch.MatchConfig()
    sec, cpu_matches, cpu_checksum = oracle.time_match_pairs(p, cfg, [d[i] for i in range(k)], [c.shorts for c in codes],
                                                              [c.longs for c in codes], pairs, os.cpu_count() or 1)
    st = matcher.match_pairs_device(pairs + BASE, cfg)
    assert st["pairs"] == 4950 and st["matches"] == cpu_matches
    assert st["records_checksum"] == cpu_checksum
    # and the host delivery of the same run carries the same records
    offs, rec, _ = matcher.match_pairs(pairs + BASE, cfg)
    assert host_checksum(offs, rec) == cpu_checksum


def test_save_matches_from_device_results(matcher, oracle, default_family, tmp_path):
    fresh(matcher, default_family)
    d = make_dataset(2, 500, seed=101)
    want = run_pair_case(matcher, oracle, default_family, d[0], d[1], [ch.MatchConfig()])
    _, rec, _ = matcher.match_pairs([(BASE, BASE + 1)], ch.MatchConfig())
    ch.save_matches("a", "b", rec, tmp_path / ch.pair_file_name(0, 1))
    oracle.save_matches("a", "b", want, tmp_path / "want.txt")
    assert (tmp_path / "match_000000_000001.txt").read_bytes() == (tmp_path / "want.txt").read_bytes()


# ---- multi-GPU host logic on the real engine (world 1; worlds 2 and 3 run under gloo on CPU) -----------
def test_sharded_job_on_device(matcher, oracle, default_family):
    from paper_1805_08995_b200.sharding import CollectingSink, Comm, ShardedJob

    fresh(matcher, default_family)
    images, points = 6, 1000
    data = make_dataset(images, points, seed=21)
    job = ShardedJob(matcher, Comm(0, 1))
    cen = job.set_centering(lambda i: data[i], images)
    matcher._test_ids |= set(range(images))
    assert np.array_equal(cen, oracle.centering([data[i] for i in range(images)]))
    pairs = ch.plan_exhaustive(images, 2, 2)
    sink = CollectingSink()
    stats = job.match(lambda i: data[i], pairs, ch.MatchConfig(), sink)
    assert (stats["first_pair"], stats["last_pair"]) == (0, len(pairs))
    counts, records = sink.result()
    offsets, recs = job.gather_results(counts, records)
    assert stats["matches"] == len(recs) == offsets[-1]
    codes = [oracle_codes(oracle, default_family, cen, data[i]) for i in range(images)]
    for k, (a, b) in enumerate(pairs):
        want, _ = oracle.match_pair(default_family.params, ch.MatchConfig(), data[a], *codes[a], data[b], *codes[b])
        assert np.array_equal(recs[offsets[k]:offsets[k + 1]], want), (k, a, b)


# ---- epipolar-guided variant (guided_match_pair, geometry.cpp:234-250) --------------
def _keypoints(n, seed, integer=False):
    rng = np.random.default_rng(seed)
    x, y = rng.uniform(0, 1000, n), rng.uniform(0, 800, n)
    if integer:
        x, y = np.floor(x), np.floor(y)
    return np.column_stack([x, y, np.full(n, 2.0), np.zeros(n)]).astype(np.float32)


@pytest.mark.parametrize("n_i,n_j,params", [(1500, 1500, ch.FamilyParams()), (900, 2100, ch.FamilyParams()),
                                             (16384, 16384, ch.FamilyParams()), (1200, 1200, ch.FamilyParams(7, 100, 5, 42)),
                                             (2000, 24577, ch.FamilyParams()), (1500, 13000, ch.FamilyParams(10, 96, 4, 99))])
def test_guided_match_bit_exact(matcher, oracle, n_i, n_j, params):
    fam = ch.build_hash_family(params)
    fresh(matcher, fam)
    desc = make_dataset(2, max(n_i, n_j), seed=31)
    d = [desc[0][:n_i], desc[1][:n_j]]
    kp = [_keypoints(n_i, 1, integer=True), _keypoints(n_j, 2)]
    for i in range(2):
        put(matcher, BASE + i, d[i], kp[i])
    matcher.centering_reset()
    matcher.centering_add(BASE)
    matcher.centering_add(BASE + 1)
    cen = matcher.centering_apply()
    matcher.hash([BASE, BASE + 1])
    codes = [oracle_codes(oracle, fam, cen, d[i]) for i in range(2)]
    rng = np.random.default_rng(5)
    F = rng.normal(size=(3, 3))
    F[:, 2] *= 300.0
    # lines degenerate exactly for the queries with x == 7 (integer query keypoints): those stay unguided
    F_some_degenerate = np.array([[1.0, 0.0, -7.0], [0.0, 0.0, 0.0], [0.0, 50.0, -20000.0]])
    cfg = ch.MatchConfig()
    base, _ = oracle.match_pair(params, cfg, d[0], *codes[0], d[1], *codes[1])
    cases = [(F, 1e9), (F, 150.0), (F, 25.0), (F, 0.0), (np.zeros((3, 3)), 4.0), (F_some_degenerate, 60.0)]
    for k, (f, band) in enumerate(cases):
        want, wstats, wranked, wcount = oracle.guided_match_pair(params, cfg, d[0], kp[0], *codes[0], d[1], kp[1], *codes[1],
                                                                 f, band, want_ranked=True)
        offs, rec, stats = matcher.match_pairs_guided([(BASE, BASE + 1)], f[None], band, cfg)
        assert np.array_equal(rec, want), (k, len(rec), len(want))
        assert stats["verified_queries"] == wstats["verified_queries"] and stats["distances"] == wstats["distances"]
        ranked, rc = matcher.ranked_guided(BASE, BASE + 1, f, band, cfg)
        assert np.array_equal(rc, wcount), k
        for q in np.flatnonzero(rc):
            assert np.array_equal(ranked[q, :rc[q]], wranked[q, :rc[q]]), (k, q)
        if k in (0, 4):  # a band that keeps everything / an all-degenerate F: plain match_pair
            assert np.array_equal(rec, base)
    assert len(oracle.guided_match_pair(params, cfg, d[0], kp[0], *codes[0], d[1], kp[1], *codes[1], F, 150.0)[0]) not in (0, len(base))
    # one call, several pairs with their own F
    offs, rec, _ = matcher.match_pairs_guided([(BASE, BASE + 1), (BASE + 1, BASE), (BASE, BASE + 1)],
                                              np.stack([F, F.T, np.zeros((3, 3))]), 150.0, cfg)
    w0, _ = oracle.guided_match_pair(params, cfg, d[0], kp[0], *codes[0], d[1], kp[1], *codes[1], F, 150.0)
    w1, _ = oracle.guided_match_pair(params, cfg, d[1], kp[1], *codes[1], d[0], kp[0], *codes[0], F.T, 150.0)
    assert np.array_equal(rec[offs[0]:offs[1]], w0) and np.array_equal(rec[offs[1]:offs[2]], w1)
    assert np.array_equal(rec[offs[2]:offs[3]], base)
    with pytest.raises(ValueError):
        matcher.match_pairs_guided([(BASE, BASE + 1)], F[None], -1.0, cfg)


def test_image_device_bytes_is_what_an_upload_takes(matcher, default_family):
    """chgpu_image_device_bytes (the device_image_bytes of chgpu_partition_sizing_for_device) against the arena's own growth."""
    fresh(matcher, default_family)
    assert matcher.image_device_bytes(0) > 0
    small, big = matcher.image_device_bytes(8192), matcher.image_device_bytes(20000)
    per_point = 128 + 16 + 16 + 6 * 4 + 6 * 2 + 6 * 2 + 6 * 34  # desc, kp, long code, short codes, points, scan, sorted copies
    assert 8192 * per_point <= small <= 8192 * per_point + 64 * 1024
    assert big > 20000 * (per_point + 6 * 4)  # + the tiles' own points / scan arrays
    with pytest.raises(ch.UnsupportedError):
        matcher.image_device_bytes(65537)


# ---- failure paths ----------------------------------------------------------------------------------
def test_failed_pair_list_leaves_the_context_usable(matcher, default_family):
    """A sink that aborts, and a record capacity that runs out, in the MIDDLE of a multi-sub-batch pair list
    (chgpu.cu run_match: the next sub-batch is already queued when the failure is seen): the call reports the failure,
    and the same context then delivers exactly the records of an undisturbed run."""
    fresh(matcher, default_family)
    n_img, n_pts = 12, 700
    ds = make_dataset(n_img, n_pts, seed=31)
    for i, d in enumerate(ds):
        put(matcher, BASE + i, d)
    ids = [BASE + i for i in range(n_img)]
    matcher.centering_reset()
    matcher.centering_add_many(ids)
    matcher.centering_apply()
    matcher.hash(ids)
    pairs = [(BASE + i, BASE + j) for i in range(n_img) for j in range(i + 1, n_img)]  # 66 pairs
    cfg = ch.MatchConfig()
    matcher.set_sub_batch_queries(5 * n_pts)  # 5 pairs per sub-batch: 14 sub-batches
    try:
        offs0, rec0, st0 = matcher.match_pairs(pairs, cfg)
        want = host_checksum(offs0, rec0)
        assert st0["match_launches"] >= 10 and len(rec0) > 0

        class Abort(Exception):
            pass

        calls = []

        def bad_sink(first, offs, rec):
            calls.append(first)
            if len(calls) == 3:
                raise Abort()

        with pytest.raises(Abort):
            matcher.match_pairs_stream(pairs, cfg, bad_sink)
        assert len(calls) == 3

        # capacity exhausted mid-list: the status says so and `total` is still the full count
        with pytest.raises(MemoryError):
            matcher.match_pairs(pairs, cfg, capacity=len(rec0) // 2)

        got = []
        matcher.match_pairs_stream(pairs, cfg, lambda first, offs, rec: got.append((first, offs.copy(), rec.copy())))
        assert [g[0] for g in got] == sorted(g[0] for g in got)
        rec = np.concatenate([g[2] for g in got])
        assert len(rec) == len(rec0) and np.array_equal(rec, rec0)
        offs1, rec1, st1 = matcher.match_pairs(pairs, cfg)
        assert np.array_equal(offs1, offs0) and np.array_equal(rec1, rec0) and host_checksum(offs1, rec1) == want
        assert st1["matches"] == st0["matches"]
    finally:
        matcher.set_sub_batch_queries(0)


def test_replaced_centering_invalidates_hashed_codes(matcher, oracle, default_family):
    """Codes hashed under one centering must not meet codes hashed under another (the reference's HashFamily is
    fixed once centered, hashing.cpp:59-64; its code caches carry the centering fingerprint): after
    chgpu_set_centering installs a different vector, images hashed before are refused until they are hashed again;
    re-installing the SAME vector changes nothing; uploaded codes are the caller's and stay valid."""
    fresh(matcher, default_family)
    ds = make_dataset(3, 300, seed=5)
    for i, d in enumerate(ds):
        put(matcher, BASE + i, d)
    ids = [BASE, BASE + 1, BASE + 2]
    cen_a = oracle.centering(list(ds))
    cen_b = cen_a + 0.25
    matcher.set_centering(cen_a)
    matcher.hash(ids)
    cfg = ch.MatchConfig()
    offs_a, rec_a, _ = matcher.match_pairs([(BASE, BASE + 1)], cfg)
    matcher.set_centering(cen_a.copy())                     # same vector: still valid
    matcher.match_pairs([(BASE, BASE + 1)], cfg)
    matcher.set_centering(cen_b)
    with pytest.raises(ch.LogicError):
        matcher.match_pairs([(BASE, BASE + 1)], cfg)
    matcher.hash([BASE])                                    # one side re-hashed is not enough
    with pytest.raises(ch.LogicError):
        matcher.match_pairs([(BASE, BASE + 1)], cfg)
    matcher.upload_codes(BASE + 2, matcher.codes(BASE + 2))  # caller-supplied codes are not tied to the centering
    matcher.match_pairs([(BASE, BASE + 2)], cfg)
    matcher.hash([BASE + 1])
    offs_b, rec_b, _ = matcher.match_pairs([(BASE, BASE + 1)], cfg)
    fam = default_family
    for k, img in enumerate((BASE, BASE + 1)):
        s, l = oracle_codes(oracle, fam, cen_b, ds[k])
        got = matcher.codes(img)
        assert np.array_equal(got.shorts, s) and np.array_equal(got.longs, l)
    matcher.set_centering(cen_a)
    matcher.hash(ids)
    offs_c, rec_c, _ = matcher.match_pairs([(BASE, BASE + 1)], cfg)
    assert np.array_equal(offs_c, offs_a) and np.array_equal(rec_c, rec_a)


# ---- threads ------------------------------------------------------------------------------------------
def test_calls_from_several_threads_on_one_context(matcher, default_family):
    """Every entry point holds the context's mutex (chgpu.cu CtxLock): W host threads that share one context — the
    reference's worker model, engine.cpp:686-696 — get serialised calls and the records of a single-threaded run."""
    import threading

    fresh(matcher, default_family)
    ds = make_dataset(6, 900, seed=55)
    for i, d in enumerate(ds):
        put(matcher, BASE + i, d)
    matcher.centering_reset()
    for i in range(6):
        matcher.centering_add(BASE + i)
    matcher.centering_apply()
    matcher.hash([BASE + i for i in range(6)])
    pairs = [(BASE + a, BASE + b) for a in range(6) for b in range(a + 1, 6)]
    cfg = ch.MatchConfig()
    want = [matcher.match_pairs([p], cfg)[1] for p in pairs]
    got = [None] * len(pairs)
    errors = []

    def worker(w):
        try:
            for rep in range(3):
                for k in range(w, len(pairs), 4):
                    got[k] = matcher.match_pairs([pairs[k]], cfg)[1]
                    matcher.codes(pairs[k][0])           # other entry points in between
                    matcher.ranked(pairs[k][0], pairs[k][1], cfg)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(w,)) for w in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k in range(len(pairs)):
        assert np.array_equal(got[k], want[k]), k
