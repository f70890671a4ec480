"""Block-pair tasks, the two-line residency schedule and the out-of-core run.

CPU part: chgpu_plan_tasks / chgpu_simulate_residency / chgpu_auto_partition_sizing (host code of libchgpu.so, no
device needed) against golden traces from the COMPILED REFERENCE (tests/golden/residency.npz), against the oracle
restatement, against the reference itself where oracle/_ref exists, and SPEC.md acceptance criterion 7
(every unordered pair exactly once; never more than 3 / 2 resident; no stall under unit cost).
GPU part: chgpu_match_plan_streamed with a handful of slots returns exactly the records of the fully resident run.
"""
import os
import struct

import numpy as np
import pytest

import paper_1805_08995_b200 as ch
from paper_1805_08995_b200 import api
from paper_1805_08995_b200.synth import make_dataset

CASES = ((10, 3, 2), (23, 2, 3), (40, 3, 4), (64, 5, 4), (9, 1, 4), (5, 8, 3), (31, 4, 1))


@pytest.fixture(scope="module")
def gold():
    from conftest import ROOT
    return np.load(ROOT / "tests" / "golden" / "residency.npz")


def task_rows(tasks):
    if not len(tasks):
        return np.zeros((0, 4), np.uint32)
    return np.stack([tasks["group_a"], tasks["group_b"], tasks["block_a"], tasks["block_b"]], 1)


def action_rows(trace):
    if not len(trace):
        return np.zeros((0, 4), np.uint32)
    return np.stack([trace["kind"], trace["level"], trace["id"], trace["prefetch"]], 1)


# ---- golden traces of the compiled reference ------------------------------------------------------------------
@pytest.mark.parametrize("case", CASES)
def test_product_equals_golden_traces(gold, case):
    k, np_, m = case
    key = f"{k}_{np_}_{m}"
    tasks = api.plan_tasks(k, np_, m)
    assert np.array_equal(task_rows(tasks), gold[f"tasks_{key}"])
    assert np.array_equal(action_rows(api.simulate_residency(tasks, api.MATCHING)), gold[f"trace_match_{key}"])
    assert np.array_equal(action_rows(api.simulate_residency(api.hashing_tasks(k, np_, m), api.HASHING)), gold[f"trace_hash_{key}"])
    acc = gold[f"accepted_{key}"]
    gt = api.plan_tasks(k, np_, m, acc)
    assert np.array_equal(task_rows(gt), gold[f"tasks_guided_{key}"])
    assert np.array_equal(action_rows(api.simulate_residency(gt, api.MATCHING)), gold[f"trace_guided_{key}"])
    # first_pair / npairs index the flat pair lists
    flat = api.plan_guided(k, np_, m, acc)
    assert int(gt["npairs"].sum()) == len(flat)
    assert np.array_equal(gt["first_pair"], np.concatenate([[0], np.cumsum(gt["npairs"])[:-1]]).astype(np.uint64))
    for t in gt:
        seg = flat[int(t["first_pair"]): int(t["first_pair"] + t["npairs"])]
        assert np.all(seg[:, 0] // np_ == t["block_a"]) and np.all(seg[:, 1] // np_ == t["block_b"])


@pytest.mark.parametrize("case", CASES)
def test_restatement_equals_golden_traces(gold, restatement, case):
    k, np_, m = case
    key = f"{k}_{np_}_{m}"
    assert np.array_equal(restatement.plan_task_blocks(k, np_, m), gold[f"tasks_{key}"])
    assert np.array_equal(restatement.simulate_residency(k, np_, m, 1), gold[f"trace_match_{key}"])
    assert np.array_equal(restatement.simulate_residency(k, np_, m, 0), gold[f"trace_hash_{key}"])
    acc = gold[f"accepted_{key}"]
    assert np.array_equal(restatement.plan_task_blocks(k, np_, m, acc), gold[f"tasks_guided_{key}"])
    assert np.array_equal(restatement.simulate_residency(k, np_, m, 1, acc), gold[f"trace_guided_{key}"])


def test_auto_partition_sizing_golden(gold, restatement):
    for (a, b), out in zip(gold["sizing_in"], gold["sizing_out"]):
        assert api.auto_partition_sizing(int(a), int(b)) == tuple(int(x) for x in out)
        assert restatement.auto_partition_sizing(int(a), int(b)) == tuple(int(x) for x in out)
    # the device rule: block_slots blocks fill the device budget, groups are whole numbers of blocks
    bi, bpg = api.partition_sizing_for_device(1_565_464, 1_179_664, 150 << 30, 1 << 40, 3, 3)
    assert 3 * bi * 1_565_464 <= 150 << 30 < 3 * (bi + 1) * 1_565_464
    assert bpg >= 1 and 3 * bpg * bi * 1_179_664 <= 1 << 40
    assert api.partition_sizing_for_device(0, 0, 0, 0, 0, 0) == (1, 1)


def test_traces_equal_reference(reference, restatement):
    rng = np.random.default_rng(5)
    for k in (1, 2, 3, 6, 11, 17, 29, 48):
        for np_ in (1, 2, 3, 5):
            for m in (1, 2, 4):
                acc = rng.integers(0, k, (2 * k, 2)).astype(np.uint32)
                acc = acc[acc[:, 0] != acc[:, 1]]
                for a in (None, acc):
                    tasks = api.plan_tasks(k, np_, m, a)
                    assert np.array_equal(task_rows(tasks), reference.plan_task_blocks(k, np_, m, a))
                    want = reference.simulate_residency(k, np_, m, 1, a)
                    assert np.array_equal(action_rows(api.simulate_residency(tasks, api.MATCHING)), want)
                    assert np.array_equal(restatement.simulate_residency(k, np_, m, 1, a), want)
                want = reference.simulate_residency(k, np_, m, 0)
                assert np.array_equal(action_rows(api.simulate_residency(api.hashing_tasks(k, np_, m), api.HASHING)), want)


# ---- SPEC.md acceptance criterion 7 + the generalised limits ------------------------------------------------------
def check_trace(tasks, trace, group_limit, block_limit):
    """Replays a trace: limits hold at every step, a task begins only with everything it needs resident, nothing a
    running task uses is evicted, tasks begin and finish in plan order, every load is used before it is evicted."""
    res = {api.GROUP: set(), api.BLOCK: set()}
    limit = {api.GROUP: group_limit, api.BLOCK: block_limit}
    running, nxt, loads = None, 0, 0
    for a in trace:
        kind, level, ident = int(a["kind"]), int(a["level"]), int(a["id"])
        if kind == api.LOAD:
            assert ident not in res[level]
            res[level].add(ident)
            assert len(res[level]) <= limit[level]
            loads += level == api.BLOCK
            if level == api.BLOCK:  # a block is parsed out of its group's bytes (engine.cpp:394-412)
                assert ident // BPG[0] in res[api.GROUP]
        elif kind == api.EVICT:
            assert ident in res[level]
            if running is not None:
                t = tasks[running]
                assert ident not in ((t["group_a"], t["group_b"]) if level == api.GROUP else (t["block_a"], t["block_b"]))
            res[level].remove(ident)
        elif kind == api.BEGIN:
            assert running is None and ident == nxt
            t = tasks[ident]
            assert {int(t["group_a"]), int(t["group_b"])} <= res[api.GROUP]
            assert {int(t["block_a"]), int(t["block_b"])} <= res[api.BLOCK]
            running = ident
        else:
            assert running == ident
            running, nxt = None, nxt + 1
    assert running is None and nxt == len(tasks)
    return loads


BPG = [1]


def test_spec_criterion_7_coverage_and_residency():
    # SPEC.md:585 asks for all K <= 64, N_p <= 5, M <= 4; the full sweep runs in seconds through the C ABI
    for k in list(range(1, 34)) + [47, 64]:
        want = {(a, b) for a in range(k) for b in range(a + 1, k)}
        for np_ in range(1, 6):
            for m in range(1, 5):
                BPG[0] = m
                tasks = api.plan_tasks(k, np_, m)
                pairs = api.plan_exhaustive(k, np_, m)
                assert int(tasks["npairs"].sum()) == len(pairs) == len(want)
                if k <= 24:
                    assert {(int(a), int(b)) for a, b in pairs} == want and len({(int(a), int(b)) for a, b in pairs}) == len(pairs)
                check_trace(tasks, api.simulate_residency(tasks, api.MATCHING), 3, 3)
                check_trace(api.hashing_tasks(k, np_, m), api.simulate_residency(api.hashing_tasks(k, np_, m), api.HASHING), 2, 2)


def test_no_stall_under_unit_cost():
    # SPEC.md:585 "no-stall": with one load per time unit and one task per time unit, a prefetching loader keeps the
    # device busy — between Begin(t) and Begin(t+1) at most the loads ONE task can hide remain on line 1.  Checked as:
    # after the first task, no task waits for more than one non-prefetch block load.
    for (k, np_, m) in ((40, 2, 3), (64, 4, 4), (33, 1, 2)):
        tasks = api.plan_tasks(k, np_, m)
        trace = api.simulate_residency(tasks, api.MATCHING)
        pending = 0
        begun = 0
        for a in trace:
            if a["kind"] == api.LOAD and a["level"] == api.BLOCK and not a["prefetch"]:
                pending += 1
            if a["kind"] == api.BEGIN:
                if begun:
                    assert pending <= 1, (k, np_, m, int(a["id"]))
                pending = 0
                begun += 1


def test_generalised_slot_limits():
    k, np_, m = 60, 2, 3
    BPG[0] = m
    tasks = api.plan_tasks(k, np_, m)
    nblocks = (k + np_ - 1) // np_
    base = check_trace(tasks, api.simulate_residency(tasks, api.MATCHING), 3, 3)
    prev = base
    for slots in (4, 6, 12, nblocks):
        trace = api.simulate_residency(tasks, api.MATCHING, group_slots=slots, block_slots=slots)
        loads = check_trace(tasks, trace, slots, slots)
        assert loads <= prev  # more room never costs loads on this plan
        prev = loads
    assert prev == nblocks  # everything fits: each block is loaded exactly once, nothing is evicted
    assert not np.any(api.simulate_residency(tasks, api.MATCHING, nblocks, nblocks)["kind"] == api.EVICT)
    # a cross task needs two blocks: one slot cannot hold it (the reference throws std::logic_error there)
    with pytest.raises(ValueError):
        api.simulate_residency(tasks, api.MATCHING, group_slots=3, block_slots=1)
    assert len(api.simulate_residency(api.plan_tasks(1, 1, 1), api.MATCHING)) == 0  # one image: no pair, no task
    with pytest.raises(ValueError):
        api.plan_tasks(0, 1, 1)
    with pytest.raises(ValueError):
        api.plan_tasks(10, 3, 2, [(1, 1)])
    with pytest.raises(ValueError):
        api.plan_tasks(10, 3, 2, [(1, 10)])
    assert len(api.plan_tasks(10, 3, 2, np.zeros((0, 2), np.uint32))) == 0


# ---- out-of-core run on the device ----------------------------------------------------------------------------
def chft_bytes(desc, kp):
    n = len(desc)
    rec = np.zeros(n, dtype=np.dtype([("kp", "<f4", 4), ("d", "u1", 128)]))
    rec["kp"], rec["d"] = kp, desc
    return b"CHFT" + struct.pack("<III", 1, n, 0) + rec.tobytes()


def write_dataset(tmp_path, sizes, seed):
    full = make_dataset(len(sizes), max(max(sizes), 1), seed=seed)
    desc = [full[k][:n] for k, n in enumerate(sizes)]
    paths = []
    for k, n in enumerate(sizes):
        kp = np.zeros((n, 4), np.float32)
        kp[:, 0] = np.arange(n) % 1000
        kp[:, 1] = np.arange(n) // 1000
        p = tmp_path / f"img{k:04d}.chft"
        p.write_bytes(chft_bytes(desc[k], kp))
        paths.append(p)
    return desc, paths


def fresh(matcher, family):
    """Drops what earlier GPU test modules left resident on the shared context and installs `family`."""
    for img in list(getattr(matcher, "_test_ids", set())):
        try:
            matcher.evict(img)
        except KeyError:
            pass
    matcher._test_ids = set()
    matcher.set_family(family)
    matcher.set_sub_batch_queries(0)


def resident_reference(matcher, desc, pairs, cfg, centering, base_id=70000):
    """The same pairs on the ordinary resident path (parity-tested against the oracle in test_gpu_parity.py)."""
    ids = [base_id + i for i in range(len(desc))]
    live = [i for i in range(len(desc)) if desc[i] is not None]
    for i in live:
        matcher.upload(ids[i], desc[i])
    matcher.set_centering(centering)
    matcher.hash([ids[i] for i in live])
    pr = np.array([(ids[a], ids[b]) for a, b in pairs], dtype=np.uint32).reshape(-1, 2)
    offs, rec, _ = matcher.match_pairs(pr, cfg)
    for i in live:
        matcher.evict(ids[i])
    return offs, rec


@pytest.mark.gpu
@pytest.mark.parametrize("guided,overlap", [(False, True), (True, True), (False, False)])
def test_streamed_run_equals_resident_run(matcher, restatement, tmp_path, monkeypatch, guided, overlap):
    if not overlap:
        monkeypatch.setenv("CHGPU_STREAM_NO_OVERLAP", "1")  # strictly in trace order
    sizes = [900, 1200, 700, 1500, 1, 1000, 0, 800, 1100, 950, 1300, 600, 1000, 1024, 990, 870, 1250, 640, 1111, 905, 1000, 333, 1500]
    desc, paths = write_dataset(tmp_path, sizes, seed=41)
    k, np_, m = len(sizes), 3, 2
    fam = ch.build_hash_family(ch.FamilyParams())
    fresh(matcher, fam)
    cfg = ch.MatchConfig()
    want_centering = restatement.centering(desc)
    centering, results = matcher.centering_pass_files(paths, block_images=4, io_threads=3)
    assert results == sizes
    assert np.array_equal(centering, want_centering)  # exact integer sums, one fp64 division per component
    acc = None
    if guided:
        rng = np.random.default_rng(3)
        acc = rng.integers(0, k, (70, 2)).astype(np.uint32)
        acc = acc[acc[:, 0] != acc[:, 1]]
    flat = api.plan_exhaustive(k, np_, m) if acc is None else api.plan_guided(k, np_, m, acc)
    got_pairs, got_counts, got_rec, got_tasks = [], [], [], []

    def sink(task, pairs, offs, rec):
        got_tasks.append(task)
        got_pairs.append(pairs)
        got_counts.append(np.diff(offs.astype(np.int64)))
        got_rec.append(rec.copy())

    stats, results = matcher.match_plan_streamed(paths, np_, m, cfg, accepted_pairs=acc, io_threads=3, sink=sink)
    assert results == sizes
    assert stats["max_resident_blocks"] <= 3 and stats["max_resident_groups"] <= 3
    assert stats["pairs"] == len(flat) and stats["pairs_skipped"] == 0
    assert got_tasks == sorted(got_tasks)
    tasks = api.plan_tasks(k, np_, m, acc)
    trace = api.simulate_residency(tasks, api.MATCHING)
    assert stats["tasks"] == len(tasks)
    assert stats["block_loads"] == int(np.sum((trace["kind"] == api.LOAD) & (trace["level"] == api.BLOCK)))
    assert stats["block_evictions"] == int(np.sum((trace["kind"] == api.EVICT) & (trace["level"] == api.BLOCK)))
    assert stats["block_loads"] > (k + np_ - 1) // np_ or guided  # blocks really were re-loaded: the run was out of core
    prefetched = int(np.sum((trace["kind"] == api.LOAD) & (trace["level"] == api.BLOCK) & (trace["prefetch"] == 1)))
    assert stats["background_block_loads"] == (prefetched if overlap else 0)  # line 2 runs behind the match calls
    assert np.array_equal(np.concatenate(got_pairs), flat)  # plan order
    # nothing is left behind on the device
    for i in range(k):
        with pytest.raises(KeyError):
            matcher.points(i)
    offs, rec = resident_reference(matcher, desc, flat, cfg, centering)
    assert np.array_equal(np.concatenate(got_counts), np.diff(offs.astype(np.int64)))
    assert np.array_equal(np.concatenate(got_rec), rec)
    assert stats["matches"] == len(rec) and len(rec) > 1000


@pytest.mark.gpu
def test_streamed_run_more_slots_and_failed_files(matcher, tmp_path):
    sizes = [800] * 14
    desc, paths = write_dataset(tmp_path, sizes, seed=43)
    good = paths[5].read_bytes()
    paths[5].write_bytes(good[: 16 + 144 * 100 + 7])  # truncated payload
    paths[9] = tmp_path / "missing.chft"
    fam = ch.build_hash_family(ch.FamilyParams())
    fresh(matcher, fam)
    cfg = ch.MatchConfig()
    centering, results = matcher.centering_pass_files(paths, block_images=5, io_threads=2)
    assert isinstance(results[5], ch.FeatureFileError) and results[5].fault == "Truncated"
    assert isinstance(results[9], ch.FeatureFileError) and results[9].fault == "MissingFile"
    assert [r for i, r in enumerate(results) if i not in (5, 9)] == [800] * 12
    k, np_, m = len(sizes), 2, 2
    flat = api.plan_exhaustive(k, np_, m)
    keep = np.array([a not in (5, 9) and b not in (5, 9) for a, b in flat])
    runs = {}
    for slots in (3, 5):
        got_pairs, got_rec = [], []
        stats, results = matcher.match_plan_streamed(paths, np_, m, cfg, group_slots=slots, block_slots=slots, io_threads=2,
                                                     sink=lambda t, p, o, r: (got_pairs.append(p), got_rec.append(r.copy())))
        assert isinstance(results[5], ch.FeatureFileError) and isinstance(results[9], ch.FeatureFileError)
        assert stats["max_resident_blocks"] <= slots
        assert stats["pairs"] == int(keep.sum()) and stats["pairs_skipped"] == int((~keep).sum())
        assert np.array_equal(np.concatenate(got_pairs), flat[keep])  # pairs of the failed images are skipped (engine.cpp:799)
        runs[slots] = (stats, np.concatenate(got_rec))
    assert np.array_equal(runs[3][1], runs[5][1])
    assert runs[5][0]["block_loads"] <= runs[3][0]["block_loads"]
    d2 = [None if i in (5, 9) else d for i, d in enumerate(desc)]
    offs, rec = resident_reference(matcher, d2, flat[keep], cfg, centering)
    assert np.array_equal(runs[3][1], rec)
    # one block slot cannot hold a cross task
    with pytest.raises(ValueError):
        matcher.match_plan_streamed(paths, np_, m, cfg, group_slots=3, block_slots=1)


@pytest.mark.gpu
def test_background_load_under_match_calls(matcher, tmp_path):
    """chgpu_load_chft_files_begin / _end: a load opened before match calls completes behind them (the calls pump it
    between sub-batches); images, per-file faults and match results are those of the blocking loader."""
    sizes = [1500, 900, 0, 2048, 700, 1200, 1, 3000, 800, 1000, 640, 5000, 900, 1100, 30, 2500]
    desc, paths = write_dataset(tmp_path, sizes, seed=47)
    paths[4] = tmp_path / "absent.chft"
    fam = ch.build_hash_family(ch.FamilyParams())
    fresh(matcher, fam)
    cfg = ch.MatchConfig()
    first, rest = list(range(0, 6)), list(range(6, len(sizes)))
    ids = [81000 + i for i in range(len(sizes))]
    res, _ = matcher.load_chft_files([paths[i] for i in first], [ids[i] for i in first], io_threads=2)
    assert isinstance(res[4], ch.FeatureFileError) and [r for i, r in enumerate(res) if i != 4] == [sizes[i] for i in first if i != 4]
    live = [i for i in first if i != 4]
    matcher.set_centering(np.full(128, 127.5))
    matcher.hash([ids[i] for i in live])
    pairs = np.array([(ids[a], ids[b]) for a in live for b in live if a < b], dtype=np.uint32)
    matcher.set_sub_batch_queries(2048)  # many sub-batches: many pumps
    try:
        want = matcher.match_pairs(pairs, cfg)
        matcher.load_chft_files_begin([paths[i] for i in rest], [ids[i] for i in rest], io_threads=3)
        with pytest.raises(ch.LogicError):
            matcher.load_chft_files([paths[0]], [99999])  # one job per context
        got = matcher.match_pairs(pairs, cfg)
        res, stats = matcher.load_chft_files_end()
    finally:
        matcher.set_sub_batch_queries(0)
    assert res == [sizes[i] for i in rest] and stats["files_ok"] == len(rest)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    for i in rest:
        d, _ = matcher.descriptors(ids[i])
        assert np.array_equal(d, desc[i])
    matcher.hash([ids[i] for i in rest])
    a, b = matcher.match_pairs([(ids[7], ids[11])], cfg)[:2]
    assert len(b) > 100
    assert matcher.load_chft_files_end() == ([], matcher.load_chft_files_end()[1])  # nothing open: a no-op
    matcher.evict_many([ids[i] for i in live + rest])
    with pytest.raises(KeyError):
        matcher.points(ids[7])


# ---- task order for descriptor reuse (CHGPU_ORDER_REUSE) ---------------------------------------------------------
def block_loads(tasks, order, slots):
    trace = api.simulate_residency(tasks[order], api.MATCHING, group_slots=max(slots, 3), block_slots=slots)
    return int(np.sum((trace["kind"] == api.LOAD) & (trace["level"] == api.BLOCK)))


def test_reuse_order_is_a_permutation_and_saves_loads_on_banded_plans():
    # a k-nearest-neighbour list (the Rome16K-shaped config): pairs (i, i + d), d <= 30, blocks of 64 images
    k, np_, m = 1024, 64, 4
    acc = np.array([(i, i + d) for i in range(k) for d in range(1, 31) if i + d < k], dtype=np.uint32)
    tasks = api.plan_tasks(k, np_, m, acc)
    nblocks = k // np_
    for slots in (3, 4, 6):
        order = api.order_tasks_for_reuse(tasks, slots)
        assert sorted(order.tolist()) == list(range(len(tasks)))
        plan_loads = block_loads(tasks, np.arange(len(tasks)), slots)
        reuse_loads = block_loads(tasks, order, slots)
        # every block once (one more where the walk starts inside the band and has to come back for the other half);
        # the reference traversal returns to blocks it has dropped
        assert nblocks <= reuse_loads <= nblocks + 1 and reuse_loads < plan_loads, (slots, reuse_loads, plan_loads)
    # exhaustive plans: never worse than the reference's serpentine on these shapes, and still a permutation
    for (k, np_, m, slots) in ((40, 4, 2, 3), (64, 4, 4, 3), (60, 5, 3, 4), (23, 2, 3, 3)):
        tasks = api.plan_tasks(k, np_, m)
        order = api.order_tasks_for_reuse(tasks, slots)
        assert sorted(order.tolist()) == list(range(len(tasks)))
        assert block_loads(tasks, order, slots) <= block_loads(tasks, np.arange(len(tasks)), slots) * 1.05
    assert len(api.order_tasks_for_reuse(api.plan_tasks(1, 1, 1), 3)) == 0


@pytest.mark.gpu
def test_streamed_run_in_reuse_order(matcher, tmp_path):
    sizes = [700 + 37 * (i % 9) for i in range(40)]
    desc, paths = write_dataset(tmp_path, sizes, seed=53)
    fam = ch.build_hash_family(ch.FamilyParams())
    fresh(matcher, fam)
    cfg = ch.MatchConfig()
    centering, _ = matcher.centering_pass_files(paths, block_images=8, io_threads=2)
    k, np_, m = len(sizes), 4, 2
    acc = np.array([(i, i + d) for i in range(k) for d in range(1, 7) if i + d < k], dtype=np.uint32)
    flat = api.plan_guided(k, np_, m, acc)
    runs = {}
    for order in (api.ORDER_REFERENCE, api.ORDER_REUSE):
        got = {}

        def sink(task, pairs, offs, rec):
            o = offs.astype(np.int64) - int(offs[0])
            for i, (a, b) in enumerate(pairs):
                got[(int(a), int(b))] = rec[o[i]:o[i + 1]].copy()

        stats, _ = matcher.match_plan_streamed(paths, np_, m, cfg, accepted_pairs=acc, io_threads=2, sink=sink, task_order=order)
        assert stats["pairs"] == len(flat) and stats["max_resident_blocks"] <= 3
        runs[order] = (stats, got)
    assert (k + np_ - 1) // np_ <= runs[api.ORDER_REUSE][0]["block_loads"] <= (k + np_ - 1) // np_ + 1
    assert runs[api.ORDER_REUSE][0]["block_loads"] < runs[api.ORDER_REFERENCE][0]["block_loads"]
    assert set(runs[0][1]) == set(runs[1][1]) == {(int(a), int(b)) for a, b in flat}
    for key, rec in runs[0][1].items():
        assert np.array_equal(rec, runs[1][1][key])
    with pytest.raises(ValueError):
        matcher.match_plan_streamed(paths, np_, m, cfg, task_order=7)


# ---- sharding a streamed run over workers (one process / context per GPU) ------------------------------------------
def test_shard_tasks_contiguous_and_balanced():
    k, np_, m = 1024, 64, 4
    acc = np.array([(i, i + d) for i in range(k) for d in range(1, 31) if i + d < k], dtype=np.uint32)
    for tasks, order in ((api.plan_tasks(k, np_, m, acc), None), (api.plan_tasks(k, np_, m, acc), "reuse"), (api.plan_tasks(48, 4, 3), None)):
        o = api.order_tasks_for_reuse(tasks, 3) if order == "reuse" else None
        seq = tasks if o is None else tasks[o]
        total = int(seq["npairs"].sum())
        for shards in (1, 2, 3, 8, len(tasks) + 5):
            first = api.shard_tasks(tasks, shards, o)
            assert first[0] == 0 and first[-1] == len(tasks) and np.all(np.diff(first.astype(np.int64)) >= 0)
            per = [int(seq["npairs"][first[i]:first[i + 1]].sum()) for i in range(shards)]
            assert sum(per) == total
            if shards <= 8:  # no worker exceeds its share by more than one task
                assert max(per) <= total / shards + int(seq["npairs"].max())
    with pytest.raises(ValueError):
        api.shard_tasks(api.plan_tasks(10, 2, 2), 0)


@pytest.mark.gpu
def test_streamed_shards_cover_the_plan(matcher, tmp_path):
    sizes = [600 + 41 * (i % 7) for i in range(24)]
    desc, paths = write_dataset(tmp_path, sizes, seed=59)
    fam = ch.build_hash_family(ch.FamilyParams())
    fresh(matcher, fam)
    cfg = ch.MatchConfig()
    matcher.centering_pass_files(paths, block_images=6, io_threads=2)
    k, np_, m = len(sizes), 3, 2
    flat = api.plan_exhaustive(k, np_, m)
    whole = {}
    matcher.match_plan_streamed(paths, np_, m, cfg, io_threads=2, task_order=api.ORDER_REUSE,
                                sink=lambda t, p, o, r: whole.update({(int(a), int(b)): r[int(o[i] - o[0]):int(o[i + 1] - o[0])].copy()
                                                                      for i, (a, b) in enumerate(p)}))
    assert set(whole) == {(int(a), int(b)) for a, b in flat}
    parts, pairs_seen = {}, 0
    for shard in range(3):  # what three GPUs would run, here one after the other on the one context
        stats, _ = matcher.match_plan_streamed(paths, np_, m, cfg, io_threads=2, task_order=api.ORDER_REUSE, shard=shard, shards=3,
                                               sink=lambda t, p, o, r: parts.update({(int(a), int(b)): r[int(o[i] - o[0]):int(o[i + 1] - o[0])].copy()
                                                                                     for i, (a, b) in enumerate(p)}))
        assert 0 < stats["pairs"] < len(flat)
        pairs_seen += stats["pairs"]
    assert pairs_seen == len(flat) and set(parts) == set(whole)  # every pair exactly once over the shards
    for key, rec in whole.items():
        assert np.array_equal(rec, parts[key])
    with pytest.raises(ValueError):
        matcher.match_plan_streamed(paths, np_, m, cfg, shard=3, shards=3)


@pytest.mark.gpu
def test_streamed_sharded_job_single_rank(matcher, restatement, tmp_path):
    from paper_1805_08995_b200.sharding import Comm, StreamedShardedJob
    sizes = [500 + 29 * (i % 5) for i in range(12)]
    desc, paths = write_dataset(tmp_path, sizes, seed=61)
    fresh(matcher, ch.build_hash_family(ch.FamilyParams()))
    job = StreamedShardedJob(matcher, Comm(0, 1))
    cen = job.set_centering(paths, block_images=5, io_threads=2)
    assert np.array_equal(cen, restatement.centering(desc))
    seen = []
    stats, results = job.match(paths, 3, 2, ch.MatchConfig(), io_threads=2, sink=lambda t, p, o, r: seen.append(p))
    assert results == sizes and stats["pairs"] == 12 * 11 // 2
    assert sorted(map(tuple, np.concatenate(seen).tolist())) == sorted(map(tuple, api.plan_exhaustive(12, 3, 2).tolist()))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", list(range(int(os.environ.get("CHSTREAM_SOAK", "4")))))
def test_streamed_run_random_partitions(matcher, tmp_path, seed):
    """Random datasets (empty, tiny, tiled images), partitions, slot limits, task orders and hash families — short codes of
    more than 12 bits and top_k > 32 (the general kernels) included: the out-of-core run delivers the records of the resident
    run, pair for pair, and leaves nothing on the device."""
    rng = np.random.default_rng(4200 + seed)
    k = int(rng.integers(5, 19))
    sizes = [int(x) for x in rng.choice([0, 1, 50, 400, 900, 1500, 2600, 12000], size=k, p=[.05, .05, .1, .2, .25, .2, .1, .05])]
    desc, paths = write_dataset(tmp_path, sizes, seed=600 + seed)
    np_, m_ = int(rng.integers(1, 5)), int(rng.integers(1, 4))
    short_bits = int(rng.choice([4, 8, 10, 14, 20]))
    fam = ch.build_hash_family(ch.FamilyParams(short_bits=short_bits, table_count=int(rng.integers(2, 9))))
    fresh(matcher, fam)
    cfg = ch.MatchConfig(top_k=int(rng.choice([2, 10, 32, 40])), hamming_threshold=int(rng.integers(30, 129)))
    centering, results = matcher.centering_pass_files(paths, block_images=int(rng.integers(1, 6)), io_threads=int(rng.integers(1, 5)))
    assert results == sizes
    acc = None
    if rng.random() < 0.4:
        acc = rng.integers(0, k, (int(rng.integers(1, 60)), 2)).astype(np.uint32)
        acc = acc[acc[:, 0] != acc[:, 1]]
        if len(acc) == 0:
            acc = None
    flat = api.plan_exhaustive(k, np_, m_) if acc is None else api.plan_guided(k, np_, m_, acc)
    slots = int(rng.choice([0, 3, 4, 6]))
    order = int(rng.choice([api.ORDER_REFERENCE, api.ORDER_REUSE]))
    got = {}

    def sink(task, pairs, offs, rec):
        o = offs.astype(np.int64)
        for i, (a, b) in enumerate(pairs):
            assert (int(a), int(b)) not in got
            got[(int(a), int(b))] = rec[o[i]: o[i + 1]].copy()

    stats, results = matcher.match_plan_streamed(paths, np_, m_, cfg, accepted_pairs=acc, group_slots=slots, block_slots=slots,
                                                 io_threads=int(rng.integers(1, 5)), sink=sink, task_order=order)
    assert stats["pairs"] == len(flat) == len(got)
    touched = {int(x) for x in np.asarray(flat).reshape(-1)}
    for i in range(k):  # (a guided plan never loads the blocks none of its pairs needs: those files report nothing)
        assert results[i] == sizes[i] or (i not in touched and results[i] == 0), (seed, i, results[i], sizes[i])
        with pytest.raises(KeyError):
            matcher.points(i)
    offs, rec = resident_reference(matcher, desc, flat, cfg, centering)
    o = offs.astype(np.int64)
    for i, (a, b) in enumerate(flat):
        assert np.array_equal(got[(int(a), int(b))], rec[o[i]: o[i + 1]]), (seed, int(a), int(b))
