"""CPU suite for the product's host side: the C-ABI library loads, exports every symbol the
header declares, and its host-only entry points (family generation, pair planning, match-file
output, sharding) agree with the oracle / golden vectors.  No device compute is called here."""
import hashlib
import re
import tempfile
from pathlib import Path

import numpy as np
import pytest

import paper_1805_08995_b200 as ch
from paper_1805_08995_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "chgpu.h").read_text()
    declared = set(re.findall(r"\b(chgpu_[a-z0-9_]+)\s*\(", header))
    declared -= {"chgpu_sink_fn"}
    lib = N.load()
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, f"libchgpu.so does not export {missing}"
    unbound = sorted(declared - set(N.SIGNATURES))
    assert not unbound, f"_native.SIGNATURES lacks {unbound}"
    assert len(declared) >= 30


def test_record_layout_is_the_reference_layout():
    import ctypes as C
    assert C.sizeof(N.MatchRecordC) == 16 and N.MatchRecordC.distance_sq.offset == 8   # feature_io.hpp:51-57
    assert ch.RECORD_DTYPE.itemsize == 16


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(ch.CudaError):
        ch.Matcher(0)


def test_family_generate_matches_golden_and_oracle(restatement, golden):
    g = golden["family"]
    for tag, params in {"default": ch.FamilyParams(), "m10_n96_L4_s99": ch.FamilyParams(10, 96, 4, 99)}.items():
        fam = ch.build_hash_family(params)
        assert sha(fam.short_planes) == str(g[tag + "_short_sha"])
        assert sha(fam.long_planes) == str(g[tag + "_long_sha"])
        sp, lp = restatement.build_family(params)
        assert np.array_equal(fam.short_planes, sp) and np.array_equal(fam.long_planes, lp)
    for bad in (ch.FamilyParams(short_bits=0), ch.FamilyParams(long_bits=8), ch.FamilyParams(long_bits=129),
                ch.FamilyParams(table_count=0)):
        with pytest.raises(ValueError):
            ch.build_hash_family(bad)


def test_plan_exhaustive_matches_golden_and_oracle(restatement, golden):
    g = golden["plans"]
    for (k, np_, m) in ((10, 3, 2), (7, 2, 2), (12, 5, 1), (9, 1, 4), (5, 8, 3)):
        assert np.array_equal(ch.plan_exhaustive(k, np_, m), g[f"pairs_{k}_{np_}_{m}"])
    for k in (1, 2, 6, 17, 40):
        for np_ in (1, 3, 4):
            for m in (1, 2, 5):
                assert np.array_equal(ch.plan_exhaustive(k, np_, m).reshape(-1, 2),
                                      restatement.plan_exhaustive(k, np_, m)[0].reshape(-1, 2))
    with pytest.raises(ValueError):
        ch.plan_exhaustive(0, 1, 1)


def test_plan_properties_at_baseline_size():
    # config 3: 1,000 images -> 499,500 pairs, every unordered pair exactly once, first < second
    pairs = ch.plan_exhaustive(1000, 50, 4)
    assert pairs.shape == (499500, 2) and (pairs[:, 0] < pairs[:, 1]).all()
    key = pairs[:, 0].astype(np.int64) * 1000 + pairs[:, 1]
    assert len(np.unique(key)) == 499500


def test_plan_guided_matches_golden_and_oracle(restatement, golden):
    g = golden["plans_guided"]
    for key in [k for k in g.files if k.startswith("accepted_")]:
        k, np_, m = (int(x) for x in key.split("_")[1:])
        assert np.array_equal(ch.plan_guided(k, np_, m, g[key]), g[f"pairs_{k}_{np_}_{m}"])
    rng = np.random.default_rng(8)
    for (k, np_, m) in ((6, 1, 1), (17, 3, 2), (40, 4, 5), (64, 64, 1)):
        acc = rng.integers(0, k, (4 * k, 2)).astype(np.uint32)
        acc = acc[acc[:, 0] != acc[:, 1]]
        assert np.array_equal(ch.plan_guided(k, np_, m, acc), restatement.plan_guided(k, np_, m, acc)[0])
        # all pairs accepted: the exhaustive plan itself
        every = ch.plan_exhaustive(k, np_, m)
        assert np.array_equal(ch.plan_guided(k, np_, m, every[rng.permutation(len(every))]), every)
    assert len(ch.plan_guided(9, 2, 2, np.zeros((0, 2), np.uint32))) == 0
    for bad in ([(3, 3)], [(0, 9)], [(12, 1)]):
        with pytest.raises(ValueError):
            ch.plan_guided(9, 2, 2, bad)


def test_plan_guided_at_config4_size_keeps_neighbours_together():
    """BASELINE config 4: 16,384 images, pairs (i, i+d), d <= 30 — planned without enumerating 134 M pairs; the plan is
    a permutation of the list in which consecutive pairs share blocks (what keeps a train image hot in shared memory)."""
    k = 16384
    acc = np.array([(i, i + d) for i in range(k) for d in range(1, 31) if i + d < k], dtype=np.uint32)
    plan = ch.plan_guided(k, 50, 4, acc)
    assert plan.shape == acc.shape == (491055, 2)
    key = lambda p: np.sort(p[:, 0].astype(np.int64) * k + p[:, 1])  # noqa: E731
    assert np.array_equal(key(plan), key(acc))
    blocks = plan // 50
    same_task = (blocks[1:] == blocks[:-1]).all(axis=1)
    assert same_task.mean() > 0.99


def test_shard_range_partitions():
    for n in (0, 1, 7, 499500):
        for world in (1, 2, 3, 8):
            spans = [ch.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_save_matches_is_byte_identical(golden, restatement):
    g = golden["small_dataset"]
    rec = g["rec_default_01"]
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "m.txt"
        ch.save_matches("img_a", "img_b", rec, p)
        assert p.read_bytes() == g["match_text_default_01"].tobytes()
        # non-integer and extreme doubles print as the shortest round-trip decimal
        odd = np.zeros(4, dtype=ch.RECORD_DTYPE)
        odd["query_index"] = [0, 1, 2, 4294967295]
        odd["train_index"] = [5, 6, 7, 8]
        odd["distance_sq"] = [0.1, 1e22, 8323200.0, 2.5e-7]
        q = Path(td) / "odd.txt"
        ch.save_matches("a", "b", odd, q)
        r = Path(td) / "odd_ref.txt"
        restatement.save_matches("a", "b", odd, r)
        assert q.read_bytes() == r.read_bytes()
        empty = Path(td) / "e.txt"
        ch.save_matches("x", "y", odd[:0], empty)
        assert empty.read_bytes() == b"# x y 0\n"
        with pytest.raises(ch.FeatureFileError):
            ch.save_matches("x", "y", odd, Path(td) / "no_such_dir" / "f.txt")
    assert ch.pair_file_name(3, 41) == "match_000003_000041.txt"      # engine.cpp:724-728
    assert ch.pair_file_name(1234567, 2) == "match_1234567_000002.txt"


# ---- work-balanced sharding (datasets of mixed image sizes) -------------------------------------------
def test_weighted_sharding_balances_work_not_pair_count():
    rng = np.random.default_rng(5)
    images = 240
    points = rng.choice(np.array([1024, 8192, 32768], dtype=np.uint32), size=images, p=[0.5, 0.4, 0.1])
    pairs = ch.plan_exhaustive(images, 16, 3)
    w = np.array([ch.pair_weight(int(points[a]), int(points[b])) for a, b in pairs], dtype=np.uint64)
    for shards in (2, 3, 4, 8):
        first, weights = ch.shard_pairs_weighted(pairs, points, shards)
        assert first[0] == 0 and first[-1] == len(pairs) and np.all(np.diff(first.astype(np.int64)) >= 0)
        mine = [int(w[int(first[s]):int(first[s + 1])].sum()) for s in range(shards)]
        assert mine == [int(x) for x in weights] and sum(mine) == int(w.sum())
        assert max(mine) / min(mine) <= 1.05, (shards, mine)
        # the pair-count split of the same list is far from balanced on this dataset
        by_count = [int(w[a:b].sum()) for a, b in (ch.shard_range(len(pairs), r, shards) for r in range(shards))]
        assert max(by_count) / min(by_count) > max(mine) / min(mine)
    # tasks: the same balance one level up (out-of-core runs shard the task sequence)
    tasks = ch.plan_tasks(images, 16, 3)
    tw = ch.task_weights(tasks, pairs, points)
    assert int(tw.sum()) == int(w.sum())
    for shards in (2, 4):
        cut = ch.shard_tasks(tasks, shards, weights=tw)
        work = [int(tw[int(cut[s]):int(cut[s + 1])].sum()) for s in range(shards)]
        plain = ch.shard_tasks(tasks, shards)
        plain_work = [int(tw[int(plain[s]):int(plain[s + 1])].sum()) for s in range(shards)]
        assert max(work) / min(work) <= max(plain_work) / min(plain_work) + 1e-9
    # uniform datasets: identical to the pair-count split up to one pair
    first, _ = ch.shard_pairs_weighted(pairs, np.full(images, 4096, np.uint32), 4)
    for r in range(4):
        a, b = ch.shard_range(len(pairs), r, 4)
        assert abs(int(first[r]) - a) <= 1 and abs(int(first[r + 1]) - b) <= 1


def test_shard_arguments_are_validated():
    with pytest.raises(ValueError):
        ch.shard_range(10, 3, 3)  # rank must be below world
    with pytest.raises(ValueError):
        ch.shard_pairs_weighted(np.array([[0, 5]], np.uint32), np.array([10, 10], np.uint32), 2)  # index beyond the image table
    with pytest.raises(ValueError):
        ch.shard_pairs_weighted(np.array([[0, 1]], np.uint32), np.array([10, 10], np.uint32), 0)
    assert ch.shard_range(10, 0, 1) == (0, 10)
