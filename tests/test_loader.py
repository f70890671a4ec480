"""Disk -> pinned host -> HBM streaming loader (chgpu_load_chft_files): every file of
a dataset written with the reference's CHFT layout arrives on the device intact, bad files are reported with
the reference's fault classes and skipped, and the fused centering pass equals the exact integer sums."""
import struct

import numpy as np
import pytest

import paper_1805_08995_b200 as ch
from paper_1805_08995_b200.synth import make_dataset

pytestmark = pytest.mark.gpu


def chft_bytes(desc, kp):
    n = len(desc)
    rec = np.zeros(n, dtype=np.dtype([("kp", "<f4", 4), ("d", "u1", 128)]))
    rec["kp"], rec["d"] = kp, desc
    return b"CHFT" + struct.pack("<III", 1, n, 0) + rec.tobytes()


@pytest.mark.parametrize("io_threads", [1, 3, 8])
def test_streaming_loader(matcher, tmp_path, io_threads):
    fam = ch.build_hash_family(ch.FamilyParams())
    for img in list(getattr(matcher, "_test_ids", set())):
        try:
            matcher.evict(img)
        except KeyError:
            pass
    matcher._test_ids = set()
    matcher.set_family(fam)
    rng = np.random.default_rng(io_threads)
    sizes = [0, 1, 700, 4096, 33, 9000, 2500, 1, 12000, 64, 5000, 300, 8192, 17, 2048, 999, 4097, 31, 20000, 7]
    full = make_dataset(len(sizes), max(sizes), seed=100)  # one dataset: the images share the twin pool
    desc = [full[k][:n] for k, n in enumerate(sizes)]
    kps = [rng.uniform(0, 1000, (n, 4)).astype(np.float32) for n in sizes]
    paths, ids = [], []
    for k, n in enumerate(sizes):
        p = tmp_path / f"img{k:03d}.chft"
        p.write_bytes(chft_bytes(desc[k], kps[k]))
        paths.append(p)
        ids.append(9000 + k)
    # faults, interleaved with good files
    good5 = paths[5].read_bytes()
    bad = {"missing": (tmp_path / "nope.chft", None), "magic": (tmp_path / "magic.chft", b"XHFT" + good5[4:]),
           "version": (tmp_path / "ver.chft", good5[:4] + struct.pack("<I", 9) + good5[8:]),
           "cut": (tmp_path / "cut.chft", good5[:16 + 144 * 100 + 5]), "tiny": (tmp_path / "tiny.chft", good5[:7])}
    for name, (p, data) in bad.items():
        if data is not None:
            p.write_bytes(data)
    order = list(zip(paths, ids))
    order.insert(3, (bad["missing"][0], 9900))
    order.insert(7, (bad["magic"][0], 9901))
    order.insert(8, (bad["version"][0], 9902))
    order.insert(15, (bad["cut"][0], 9903))
    order.append((bad["tiny"][0], 9904))
    matcher.centering_reset()
    results, stats = matcher.load_chft_files([p for p, _ in order], [i for _, i in order], io_threads=io_threads,
                                             accumulate_centering=True)
    matcher._test_ids |= set(ids)
    want_fault = {9900: ("MissingFile", 0), 9901: ("BadMagic", 0), 9902: ("BadVersion", 4),
                  9903: ("Truncated", 16 + 144 * 100 + 5), 9904: ("Truncated", 7)}
    for (p, i), r in zip(order, results):
        if i in want_fault:
            assert isinstance(r, ch.FeatureFileError) and (r.fault, r.byte_offset) == want_fault[i], (p.name, r)
            with pytest.raises(KeyError):
                matcher.points(i)
        else:
            assert r == sizes[i - 9000], p.name
    assert stats["files_ok"] == len(sizes) and stats["files_failed"] == 5 and stats["points"] == sum(sizes)
    for k, n in enumerate(sizes):
        d, kp = matcher.descriptors(9000 + k)
        assert np.array_equal(d, desc[k]) and np.array_equal(kp, kps[k]), k
    sums, count = matcher.centering_sums()
    assert count == sum(sizes)
    assert np.array_equal(sums, sum(d.astype(np.uint64).sum(0) for d in desc))
    # the loaded images hash and match like uploaded ones
    matcher.centering_apply()
    matcher.hash([9003, 9012])
    a = matcher.match_pairs([(9003, 9012)])[1]
    matcher.upload(9500, desc[3], kps[3])
    matcher.upload(9501, desc[12], kps[12])
    matcher._test_ids |= {9500, 9501}
    matcher.hash([9500, 9501])
    b = matcher.match_pairs([(9500, 9501)])[1]
    assert np.array_equal(a, b) and len(a) > 0
