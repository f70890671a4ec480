"""Generates tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref/libcashash_ref.so, i.e. the
reference's own translation units built in place from /root/reference/proj/src — see oracle/Makefile).

Run in the build container only (the GPU box has no /root/reference):
    make -C oracle ref && python tests/golden/make_golden.py
The fixtures pin the oracle restatement and the CUDA path on machines where the reference itself
cannot be built.
"""
from __future__ import annotations

import hashlib
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib  # noqa: E402
from paper_1805_08995_b200.api import FamilyParams, MatchConfig  # noqa: E402
from paper_1805_08995_b200.synth import make_dataset  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    ref = oracle_lib.reference()
    if ref is None:
        raise SystemExit("oracle/_ref/libcashash_ref.so missing: run `make -C oracle ref` first")
    assert ref.name == "reference"

    # ---- family ---------------------------------------------------------------------------------
    fam = {}
    for tag, params in {"default": FamilyParams(), "m10_n96_L4_s99": FamilyParams(10, 96, 4, 99)}.items():
        sp, lp = ref.build_family(params)
        fam[tag + "_short_sha"] = sha(sp)
        fam[tag + "_long_sha"] = sha(lp)
        fam[tag + "_short_head"] = sp[:2, :4].copy()
        fam[tag + "_long_tail"] = lp[-1, -4:].copy()
    fam["mix64_1_2_3"] = np.uint64(ref.mix64(1, 2, 3))
    fam["mix64_seed1_long_5"] = np.uint64(ref.mix64(1, 0xffffffff, 5))
    np.savez(OUT / "family.npz", **fam)

    # ---- one small dataset, every intermediate artefact -------------------------------------------
    params = FamilyParams()
    sp, lp = ref.build_family(params)
    desc = make_dataset(3, 300, seed=11, rho=0.3, sigma=8.0)
    centering = ref.centering([desc[0], desc[1], desc[2]])
    out = {"desc": desc, "centering": centering}
    codes = []
    for i in range(3):
        for rr in (3, 0, 7):
            s, l = ref.compute_codes(params, sp, lp, centering, desc[i], rr)
            if rr == 3:
                codes.append((s, l))
                out[f"shorts{i}"], out[f"longs{i}"] = s, l
            else:
                out[f"shorts{i}_rr{rr}_sha"], out[f"longs{i}_rr{rr}_sha"] = sha(s), sha(l)
    offs, pts = ref.build_bucket_index(params.short_bits, params.table_count, codes[1][0])
    out["offs1"], out["pts1"] = offs, pts
    cfgs = {
        "default": MatchConfig(),
        "tau128": MatchConfig(hamming_threshold=128),
        "k2_min5": MatchConfig(top_k=2, min_candidates_for_ratio=5),
        "tau60_k32_r09": MatchConfig(top_k=32, hamming_threshold=60, ratio=0.9),
        "tau0": MatchConfig(hamming_threshold=0),
    }
    for tag, cfg in cfgs.items():
        for (a, b) in ((0, 1), (1, 2), (2, 0)):
            rec, stats, ranked, rcount = ref.match_pair(params, cfg, desc[a], *codes[a], desc[b], *codes[b],
                                                        want_ranked=True)
            out[f"rec_{tag}_{a}{b}"] = rec
            out[f"ranked_{tag}_{a}{b}"] = ranked
            out[f"rcount_{tag}_{a}{b}"] = rcount
            out[f"stats_{tag}_{a}{b}"] = np.array(list(stats.values()), dtype=np.uint64)
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "m.txt"
        ref.save_matches("img_a", "img_b", out["rec_default_01"], p)
        out["match_text_default_01"] = np.frombuffer(p.read_bytes(), dtype=np.uint8)
    out["brute_01"] = ref.brute_force_match(desc[0], desc[1], 0.8)
    np.savez_compressed(OUT / "small_dataset.npz", **out)

    # ---- scheduler ------------------------------------------------------------------------------
    plans = {}
    for (k, np_, m) in ((10, 3, 2), (7, 2, 2), (12, 5, 1), (9, 1, 4), (5, 8, 3)):
        pairs, sizes = ref.plan_exhaustive(k, np_, m)
        plans[f"pairs_{k}_{np_}_{m}"] = pairs
        plans[f"sizes_{k}_{np_}_{m}"] = sizes
    np.savez_compressed(OUT / "plans.npz", **plans)
    # plan_guided (scheduler.cpp:144-164) on seeded accepted lists: swapped pairs and duplicates included
    guided = {}
    rng = np.random.default_rng(17)
    for (k, np_, m, cnt) in ((10, 3, 2, 12), (23, 4, 2, 60), (40, 5, 3, 200), (9, 1, 4, 36)):
        acc = rng.integers(0, k, (cnt, 2)).astype(np.uint32)
        acc = acc[acc[:, 0] != acc[:, 1]]
        acc = np.concatenate([acc, acc[:3, ::-1], acc[:2]])
        pairs, sizes = ref.plan_guided(k, np_, m, acc)
        guided[f"accepted_{k}_{np_}_{m}"] = acc
        guided[f"pairs_{k}_{np_}_{m}"] = pairs
        guided[f"sizes_{k}_{np_}_{m}"] = sizes
    np.savez_compressed(OUT / "plans_guided.npz", **guided)
    # ---- residency schedule (scheduler.cpp:175-345): task blocks and full action traces -----------------------------
    res = {}
    rng = np.random.default_rng(29)
    for (k, np_, m) in ((10, 3, 2), (23, 2, 3), (40, 3, 4), (64, 5, 4), (9, 1, 4), (5, 8, 3), (31, 4, 1)):
        key = f"{k}_{np_}_{m}"
        res[f"tasks_{key}"] = ref.plan_task_blocks(k, np_, m)
        res[f"trace_match_{key}"] = ref.simulate_residency(k, np_, m, 1)
        res[f"trace_hash_{key}"] = ref.simulate_residency(k, np_, m, 0)
        acc = rng.integers(0, k, (3 * k, 2)).astype(np.uint32)
        acc = acc[acc[:, 0] != acc[:, 1]]
        res[f"accepted_{key}"] = acc
        res[f"tasks_guided_{key}"] = ref.plan_task_blocks(k, np_, m, acc)
        res[f"trace_guided_{key}"] = ref.simulate_residency(k, np_, m, 1, acc)
    sizing_in = np.array([[1179664, 64 << 30], [0, 0], [1, 10], [1565464, 180 << 30], [144, 1 << 20], [10**6, 10**6]], dtype=np.uint64)
    res["sizing_in"] = sizing_in
    res["sizing_out"] = np.array([ref.auto_partition_sizing(int(a), int(b)) for a, b in sizing_in], dtype=np.uint32)
    np.savez_compressed(OUT / "residency.npz", **res)
    # ---- code cache written by the reference (hashing.cpp:184-206) for image 0 of the small dataset --
    cache = {"centering_fp": np.uint64(ref.centering_fingerprint(centering))}
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "c.chcc"
        ref.save_code_cache(params, int(cache["centering_fp"]), codes[0][0], codes[0][1], p)
        cache["chcc_image0"] = np.frombuffer(p.read_bytes(), dtype=np.uint8)
    np.savez_compressed(OUT / "cache.npz", **cache)
    print("wrote", [p.name for p in OUT.glob("*.npz")])


if __name__ == "__main__":
    main()
