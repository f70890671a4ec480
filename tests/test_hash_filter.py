"""Hash build through the filters (K1f fp32 SIMT, hash_kernels.cuh; K1t tensor cores / tcgen05 int8 limbs, hash_tc.cuh)
versus the exact fp64 kernel and the CPU oracle.

The filter proves most hyperplane signs from an fp32 contraction and an a-priori error bound; every dot it
cannot decide is re-evaluated in the reference's fp64 operation order (reduce_dot, hashing.hpp:24-43).  Codes
must be bit-exact in both modes, for benign and for adversarial inputs (dots at or near zero, queue overflow,
centerings outside the bound's premises)."""
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


@pytest.fixture(params=[0, 2], ids=["fp32_filter", "tensor_filter"])
def mode(request, matcher):
    """Every test runs under both filters; the context goes back to the default afterwards."""
    yield request.param
    matcher.set_hash_mode(2)  # the context's default


def install(matcher, fam, mode=0):
    for img in list(getattr(matcher, "_test_ids", set())):
        try:
            matcher.evict(img)
        except KeyError:
            pass
    matcher._test_ids = set()
    matcher.set_family(fam)
    matcher.set_hash_mode(mode)


def put(matcher, image_id, desc):
    matcher.upload(image_id, desc)
    matcher._test_ids.add(image_id)


def check(matcher, oracle, fam, cen, descs, rrs=(3,)):
    for rr in rrs:
        matcher.hash([BASE + i for i in range(len(descs))], rr)
        for i, d in enumerate(descs):
            s, l = oracle.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, d, rr)
            c = matcher.codes(BASE + i)
            assert np.array_equal(c.shorts, s), (rr, i)
            assert np.array_equal(c.longs, l), (rr, i)


@pytest.mark.parametrize("params", [ch.FamilyParams(), ch.FamilyParams(12, 128, 8, 3), ch.FamilyParams(5, 33, 7, 4)])
def test_filtered_and_exact_modes_agree_with_the_oracle(matcher, oracle, params, mode):
    fam = ch.build_hash_family(params)
    install(matcher, fam, mode)
    descs = list(make_dataset(3, 3000, seed=31)) + [make_dataset(1, 777, seed=32, shape="sift")[0]]
    cen = oracle.centering(descs)
    matcher.set_centering(cen)
    for i, d in enumerate(descs):
        put(matcher, BASE + i, d)
    before = matcher.hash_stats()
    assert before["filter_active"] == 1
    check(matcher, oracle, fam, cen, descs, rrs=(3, 0, 7))
    after = matcher.hash_stats()
    dots = 3 * sum(len(d) for d in descs) * (params.table_count * params.short_bits + params.long_bits)
    undecided = after["undecided_dots"] - before["undecided_dots"]
    assert 0 < undecided < dots * 1e-3, (undecided, dots)   # the bound is tight enough to be useful
    assert after["overflowed_batches"] == before["overflowed_batches"]
    filtered = [matcher.codes(BASE + i) for i in range(len(descs))]
    matcher.set_hash_mode(True)
    try:
        assert matcher.hash_stats()["filter_active"] == 0
        matcher.hash([BASE + i for i in range(len(descs))], 3)
        for i in range(len(descs)):
            c = matcher.codes(BASE + i)
            assert np.array_equal(c.shorts, filtered[i].shorts) and np.array_equal(c.longs, filtered[i].longs)
        assert matcher.hash_stats()["undecided_dots"] == after["undecided_dots"]
    finally:
        matcher.set_hash_mode(mode)


def test_dots_at_and_near_zero_go_to_the_exact_path(matcher, oracle, mode):
    """Descriptors at / next to an integer centering: every dot is 0 or tiny, far below the fp32 bound."""
    fam = ch.build_hash_family(ch.FamilyParams())
    install(matcher, fam, mode)
    rng = np.random.default_rng(3)
    cen = rng.integers(40, 200, 128).astype(np.float64)
    d = np.tile(cen.astype(np.uint8), (2000, 1))
    for p in range(1, 2000):   # row 0 stays exactly at the centering: all dots == 0 -> all bits 0
        k = rng.integers(1, 4)
        idx = rng.choice(128, k, replace=False)
        d[p, idx] = np.clip(d[p, idx].astype(np.int64) + rng.integers(-1, 2, k), 0, 255)
    matcher.set_centering(cen)
    put(matcher, BASE, d)
    before = matcher.hash_stats()
    check(matcher, oracle, fam, cen, [d], rrs=(3, 0, 5, 7))
    c = matcher.codes(BASE)
    assert not c.shorts[0].any() and not c.longs[0].any()
    after = matcher.hash_stats()
    # |dot| is 0 or a few |h_x|: a good part of them sits below the fp32 bound (~0.1 here); the integer filter's bound is
    # ~45x tighter and keeps little more than the exact zeros (row 0: 176 dots in each of the 4 runs)
    undecided = after["undecided_dots"] - before["undecided_dots"]
    assert undecided > (4 * 2000 * 176 * 0.1 if mode == 0 else 4 * 176 - 1)
    # a fractional centering that puts dots within 1e-9 of zero
    cen2 = cen + 1e-9
    matcher.set_centering(cen2)
    check(matcher, oracle, fam, cen2, [d])


def test_queue_overflow_falls_back_to_the_exact_kernel(matcher, oracle, mode):
    fam = ch.build_hash_family(ch.FamilyParams())
    install(matcher, fam, mode)
    cen = np.full(128, 100.0)
    n = 16384   # 16384 x 176 undecided dots > the 2^21-entry queue
    d = np.full((n, 128), 100, np.uint8)
    d[::7] = make_dataset(1, len(d[::7]), seed=9)[0]
    matcher.set_centering(cen)
    put(matcher, BASE, d)
    before = matcher.hash_stats()
    check(matcher, oracle, fam, cen, [d])
    after = matcher.hash_stats()
    assert after["overflowed_batches"] == before["overflowed_batches"] + 1


def test_centering_outside_the_bound_premises_uses_the_exact_kernel(matcher, oracle, mode):
    fam = ch.build_hash_family(ch.FamilyParams())
    install(matcher, fam, mode)
    d = make_dataset(1, 1000, seed=11)[0]
    cen = oracle.centering([d])
    cen[5] = 3e7
    matcher.set_centering(cen)
    assert matcher.hash_stats()["filter_active"] == 0
    put(matcher, BASE, d)
    check(matcher, oracle, fam, cen, [d])
    matcher.set_centering(oracle.centering([d]))
    assert matcher.hash_stats()["filter_active"] == 1


def test_more_images_than_one_hash_launch_holds(matcher, oracle, mode):
    """The filtered path hashes in launches of <= 2,048 images (one undecided-dot queue per launch)."""
    fam = ch.build_hash_family(ch.FamilyParams())
    install(matcher, fam, mode)
    k = 2300
    d = make_dataset(k, 24, seed=77)
    cen = oracle.centering(list(d))
    matcher.set_centering(cen)
    ids = [BASE + i for i in range(k)]
    matcher.upload_many(ids, np.ascontiguousarray(d))
    matcher._test_ids.update(ids)
    matcher.hash(ids)
    for i in (0, 1, 2047, 2048, 2049, k - 1):
        s, l = oracle.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, d[i])
        c = matcher.codes(ids[i])
        assert np.array_equal(c.shorts, s) and np.array_equal(c.longs, l), i
