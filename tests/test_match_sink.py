"""Asynchronous batched match-file writer: the files equal the reference's save_matches
output byte for byte, whatever the number of writer threads, and a failing file never stops the batch."""
import numpy as np
import pytest

import oracle_lib
import paper_1805_08995_b200 as ch
from paper_1805_08995_b200.synth import make_dataset


def fake_results(npairs, seed):
    rng = np.random.default_rng(seed)
    pairs = np.array([(a, b) for a in range(40) for b in range(a + 1, 40)][:npairs], dtype=np.uint32)
    counts = rng.integers(0, 60, npairs)
    counts[3] = 0
    offsets = np.zeros(npairs + 1, dtype=np.uint64)
    np.cumsum(counts, out=offsets[1:])
    rec = np.zeros(int(offsets[-1]), dtype=ch.RECORD_DTYPE)
    rec["query_index"] = rng.integers(0, 8192, len(rec))
    rec["train_index"] = rng.integers(0, 8192, len(rec))
    rec["distance_sq"] = rng.integers(0, 8323200, len(rec)).astype(np.float64)
    rec["distance_sq"][::7] += 0.5  # non-integers print with a decimal point
    return pairs, offsets, rec


@pytest.mark.parametrize("threads", [1, 4])
def test_sink_files_are_byte_identical(tmp_path, threads):
    orc = oracle_lib.best()
    names = [f"img_{k:04d}" for k in range(40)]
    pairs, offsets, rec = fake_results(300, threads)
    out = tmp_path / "out"
    out.mkdir()
    sink = ch.MatchFileSink(out, names, threads=threads, max_queued_batches=2)
    for lo in range(0, 300, 64):  # sub-batches, offsets relative to the whole record array
        hi = min(300, lo + 64)
        sink.accept(pairs[lo:hi], offsets[lo:hi + 1], rec)
    stats = sink.close()
    assert stats["files_written"] == 300 and stats["files_failed"] == 0 and stats["records"] == len(rec)
    ref = tmp_path / "ref.txt"
    total = 0
    for k, (a, b) in enumerate(pairs):
        f = out / ch.pair_file_name(int(a), int(b))
        orc.save_matches(names[a], names[b], rec[offsets[k]:offsets[k + 1]], ref)
        assert f.read_bytes() == ref.read_bytes(), k
        total += f.stat().st_size
    assert stats["bytes"] == total
    assert len(list(out.iterdir())) == 300


def test_sink_counts_failures_and_default_names(tmp_path):
    pairs, offsets, rec = fake_results(10, 9)
    sink = ch.MatchFileSink(tmp_path / "missing_dir", None, threads=2)
    sink.accept(pairs, offsets, rec)
    stats = sink.close()
    assert stats["files_written"] == 0 and stats["files_failed"] == 10
    sink = ch.MatchFileSink(tmp_path, None, threads=2)
    sink.accept(pairs[:1], offsets[:2], rec)
    assert sink.close()["files_written"] == 1
    first = (tmp_path / ch.pair_file_name(int(pairs[0][0]), int(pairs[0][1]))).read_text().splitlines()[0]
    assert first == f"# {pairs[0][0]} {pairs[0][1]} {int(offsets[1])}"


@pytest.mark.gpu
def test_match_pairs_to_files(matcher, tmp_path):
    orc = oracle_lib.best()
    fam = ch.build_hash_family(ch.FamilyParams())
    for img in list(getattr(matcher, "_test_ids", set())):
        try:
            matcher.evict(img)
        except KeyError:
            pass
    matcher._test_ids = set()
    matcher.set_family(fam)
    matcher.set_sub_batch_queries(3000)  # several sub-batches
    images = 6
    data = make_dataset(images, 1000, seed=13)
    matcher.centering_reset()
    for i in range(images):
        matcher.upload(8000 + i, data[i])
        matcher._test_ids.add(8000 + i)
        matcher.centering_add(8000 + i)
    cen = matcher.centering_apply()
    ids = np.arange(8000, 8000 + images, dtype=np.uint32)
    matcher.hash(ids)
    pairs = ch.plan_exhaustive(images, 2, 2) + 8000
    names = {8000 + i: f"scene/{i}" for i in range(images)}
    sink = ch.MatchFileSink(tmp_path, [names.get(k, str(k)) for k in range(8000 + images)], threads=3)
    st = matcher.match_pairs_to_files(pairs, sink)
    stats = sink.close()
    matcher.set_sub_batch_queries(0)
    assert stats["files_written"] == len(pairs) and stats["records"] == st["matches"]
    codes = [orc.compute_codes(fam.params, fam.short_planes, fam.long_planes, cen, data[i]) for i in range(images)]
    ref = tmp_path / "ref.txt"
    for a, b in pairs:
        want, _ = orc.match_pair(fam.params, ch.MatchConfig(), data[a - 8000], *codes[a - 8000], data[b - 8000], *codes[b - 8000])
        orc.save_matches(names[int(a)], names[int(b)], want, ref)
        assert (tmp_path / ch.pair_file_name(int(a), int(b))).read_bytes() == ref.read_bytes()
