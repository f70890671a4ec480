"""CHCC code caches and CHCV centering files: the files this library writes are
byte-identical to the reference's (hashing.cpp:184-206) and each side loads the other's, with the
reference's fault classes and offsets (hashing.cpp:228-272)."""
import numpy as np
import pytest

import oracle_lib
import paper_1805_08995_b200 as ch
from paper_1805_08995_b200.synth import make_dataset


def checkers():
    out = [oracle_lib.restatement()]
    if oracle_lib.reference() is not None:
        out.append(oracle_lib.reference())
    return out


@pytest.fixture(scope="module")
def sample(restatement):
    params = ch.FamilyParams(7, 100, 5, 42)
    fam = ch.build_hash_family(params)
    desc = make_dataset(2, 257, seed=3)
    cen = restatement.centering([desc[0], desc[1]])
    shorts, longs = restatement.compute_codes(params, fam.short_planes, fam.long_planes, cen, desc[0])
    return params, cen, ch.ImageCodes(params, shorts, longs)


def test_fingerprint_equals_checkers(sample, golden):
    _, cen, _ = sample
    for orc in checkers():
        assert ch.centering_fingerprint(cen) == orc.centering_fingerprint(cen)
        assert ch.centering_fingerprint(np.zeros(128)) == orc.centering_fingerprint(np.zeros(128))
    assert ch.centering_fingerprint(golden["small_dataset"]["centering"]) == int(golden["cache"]["centering_fp"])


def test_cache_equals_golden_bytes(golden, tmp_path, restatement):
    """The reference's own CHCC file for image 0 of the golden dataset (tests/golden/make_golden.py)."""
    g, c = golden["small_dataset"], golden["cache"]
    codes = ch.ImageCodes(ch.FamilyParams(), g["shorts0"], g["longs0"])
    f = tmp_path / "c.chcc"
    ch.save_code_cache(codes, int(c["centering_fp"]), f)
    assert f.read_bytes() == c["chcc_image0"].tobytes()
    restatement.save_code_cache(ch.FamilyParams(), int(c["centering_fp"]), g["shorts0"], g["longs0"], f)
    assert f.read_bytes() == c["chcc_image0"].tobytes()


def test_cache_files_are_byte_identical_and_cross_load(sample, tmp_path):
    params, cen, codes = sample
    fp = ch.centering_fingerprint(cen)
    ours = tmp_path / "ours.chcc"
    ch.save_code_cache(codes, fp, ours)
    assert ours.stat().st_size == 44 + 257 * 5 * 4 + 257 * 16
    for orc in checkers():
        theirs = tmp_path / f"{orc.name}.chcc"
        orc.save_code_cache(params, fp, codes.shorts, codes.longs, theirs)
        assert ours.read_bytes() == theirs.read_bytes()
        back = ch.load_code_cache(theirs, params, fp)  # we read the checker's file
        assert np.array_equal(back.shorts, codes.shorts) and np.array_equal(back.longs, codes.longs)
        s, l, fault, _ = orc.load_code_cache(ours, params, fp, 257)  # the checker reads ours
        assert fault == 0 and np.array_equal(s, codes.shorts) and np.array_equal(l, codes.longs)
    assert ch.read_code_cache_header(ours) == (params, fp, 257)


def test_cache_faults_follow_the_reference(sample, tmp_path):
    params, cen, codes = sample
    fp = ch.centering_fingerprint(cen)
    good = tmp_path / "good.chcc"
    ch.save_code_cache(codes, fp, good)
    blob = good.read_bytes()

    def variants():
        yield "missing", None, tmp_path / "nope.chcc"
        for name, data in (("magic", b"XHCC" + blob[4:]), ("short_header", blob[:20]), ("version", blob[:4] + b"\x02\0\0\0" + blob[8:]),
                           ("cut_shorts", blob[:44 + 100]), ("cut_longs", blob[:-3]), ("empty", b"")):
            p = tmp_path / f"{name}.chcc"
            p.write_bytes(data)
            yield name, data, p

    for name, data, path in variants():
        wants = [orc.load_code_cache(path, params, fp, 257)[2:] for orc in checkers()]
        assert all(w == wants[0] for w in wants), name
        fault, off = wants[0]
        assert fault != 0, name
        with pytest.raises(ch.FeatureFileError) as e:
            ch.load_code_cache(path, params, fp)
        assert (e.value.fault, e.value.byte_offset) == (ch.FeatureFileError.FAULTS[fault], off), name
        if name in ("missing", "magic", "short_header", "version", "empty"):
            assert ch.read_code_cache_header(path) is None  # hashing.cpp:208-226 returns false

    # echoed parameters or fingerprint differ: std::runtime_error in the reference
    for other, ofp in ((ch.FamilyParams(7, 100, 5, 43), fp), (params, fp ^ 1)):
        for orc in checkers():
            assert orc.load_code_cache(good, other, ofp, 257)[2] == 6
        with pytest.raises(ch.CacheMismatchError):
            ch.load_code_cache(good, other, ofp)
    with pytest.raises(ch.FeatureFileError):
        ch.save_code_cache(codes, fp, tmp_path / "no_dir" / "x.chcc")


def test_centering_file_round_trip(sample, tmp_path):
    params, cen, _ = sample
    f = tmp_path / "centering.chcv"
    ch.save_centering_file(f, params, cen)
    raw = f.read_bytes()
    # engine.cpp:522-541: "CHCV", u32 1, m, n, L, u64 seed, 128 doubles
    assert len(raw) == 28 + 1024 and raw[:4] == b"CHCV"
    assert np.array_equal(np.frombuffer(raw[4:20], dtype="<u4"), [1, 7, 100, 5])
    assert int(np.frombuffer(raw[20:28], dtype="<u8")[0]) == 42
    assert np.array_equal(np.frombuffer(raw[28:], dtype="<f8"), cen)
    p2, c2 = ch.load_centering_file(f)
    assert p2 == params and np.array_equal(c2, cen)
    with pytest.raises(ch.FeatureFileError):
        ch.load_centering_file(tmp_path / "absent.chcv")


@pytest.mark.gpu
def test_device_caches_resume_the_hash_stage(matcher, tmp_path):
    """run_hash's resume path (engine.cpp:575-582): codes written once are installed instead of recomputed."""
    orc = oracle_lib.best()
    fam = ch.build_hash_family(ch.FamilyParams())
    for img in list(getattr(matcher, "_test_ids", set())):
        try:
            matcher.evict(img)
        except KeyError:
            pass
    matcher._test_ids = set()
    matcher.set_family(fam)
    desc = make_dataset(2, 1500, seed=5)
    for i in range(2):
        matcher.upload(7000 + i, desc[i])
        matcher._test_ids.add(7000 + i)
    matcher.centering_reset()
    matcher.centering_add(7000)
    matcher.centering_add(7001)
    cen = matcher.centering_apply()
    matcher.hash([7000, 7001])
    want = [matcher.codes(7000 + i) for i in range(2)]
    _, rec0, _ = matcher.match_pairs([(7000, 7001)])
    files = [tmp_path / f"{i}.chcc" for i in range(2)]
    for i in range(2):
        matcher.save_code_cache(7000 + i, files[i])
        s, l, fault, _ = orc.load_code_cache(files[i], fam.params, orc.centering_fingerprint(cen), 1500)
        assert fault == 0 and np.array_equal(s, want[i].shorts) and np.array_equal(l, want[i].longs)
    # fresh upload (codes invalid), then install the caches: matching works without hashing
    for i in range(2):
        matcher.upload(7000 + i, desc[i])
        with pytest.raises(ch.LogicError):
            matcher.codes(7000 + i)
        matcher.load_code_cache(7000 + i, files[i])
        got = matcher.codes(7000 + i)
        assert np.array_equal(got.shorts, want[i].shorts) and np.array_equal(got.longs, want[i].longs)
    _, rec1, _ = matcher.match_pairs([(7000, 7001)])
    assert np.array_equal(rec0, rec1) and len(rec1) > 0
    # a cache for another point count or another centering is refused
    matcher.upload(7002, desc[0][:100])
    matcher._test_ids.add(7002)
    with pytest.raises(ch.CacheMismatchError):
        matcher.load_code_cache(7002, files[0])
    matcher.set_centering(np.zeros(128))
    with pytest.raises(ch.CacheMismatchError):
        matcher.load_code_cache(7000, files[0])
    with pytest.raises(ch.FeatureFileError):
        matcher.load_code_cache(7000, tmp_path / "absent.chcc")
