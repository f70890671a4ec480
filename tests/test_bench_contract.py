"""bench.py's reference arm (CPU, no GPU needed) keeps the driver's JSON contract, and `--gpus N` is a real N-rank,
strong-scaled run: launched by bench.py itself, the ONE pair list sharded, n_gpus = the ranks that ran."""
import io
import json
import subprocess
import sys
from contextlib import redirect_stdout
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
SMALL = ["--images", "9", "--points", "320", "--block-images", "3", "--blocks-per-group", "2", "--steps", "1", "--warmup", "3",
         "--e2e-steps", "1", "--no-cpu"]


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--images", "12", "--points", "512",
                        "--block-images", "4", "--blocks-per-group", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "pairs/s" and d["higher_is_better"] is True
    assert d["metric"].startswith("image pairs matched/sec") and d["value"] > 0 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] == d["e2e"]["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"] and "model" not in d["config"]


def run_ranks(world: int, extra=()):
    import bench
    argv = ["--gpus", str(world), *SMALL, *extra]
    cmd = [sys.executable, "-c",
           "import sys; sys.path.insert(0, %r); import bench; sys.exit(bench.spawn_ranks(%d, %r, script=%r, check_devices=False))"
           % (str(ROOT), world, argv, str(ROOT / "tests" / "bench_worker.py"))]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_gpus_n_is_a_strong_scaled_run_of_one_pair_list():
    """World 2 through bench.py's own launcher and main() (oracle-backed engine stand-in, gloo): the JSON line reports the
    ranks that ran, strong scaling, per-rank timings, and the shards together are the one pair list."""
    one = run_ranks(1)
    two = run_ranks(2)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["scaling"] == "strong" and two["config"]["pairs_per_step"] == 36 == one["config"]["pairs_per_step"]
    assert len(two["ranks"]) == 2 and [r["rank"] for r in two["ranks"]] == [0, 1]
    assert sum(r["pairs"] for r in two["ranks"]) == 36          # every pair exactly once over the ranks
    assert two["matches_per_step"] == one["matches_per_step"]   # worker invariance
    assert len({r["centering_fingerprint"] for r in two["ranks"]}) == 1
    assert two["ranks"][0]["centering_fingerprint"] == one["ranks"][0]["centering_fingerprint"]
    assert two["shard_work"]["max_over_min"] <= 1.2 and two["ms_per_step"] >= max(r["ms_per_step"] for r in two["ranks"]) - 1e-6
    assert two["e2e"]["value"] > 0 and two["e2e"]["h2d_bytes_per_step"] > 0 and two["gpu_launches"] == 6
    assert all(r["images_resident"] <= 9 for r in two["ranks"])


def test_gpus_must_agree_with_the_launcher_and_the_box(monkeypatch, capsys):
    import bench
    # a torchrun launch of another size than --gpus is refused instead of reporting the wrong n_gpus
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setenv("RANK", "0")
    assert bench.main(["--gpus", "2", *SMALL]) == 2
    assert "must agree" in capsys.readouterr().err
    # no launcher and fewer devices than asked for (this container has none): loud failure, nothing timed
    monkeypatch.delenv("WORLD_SIZE")
    import torch
    if (torch.cuda.device_count() if torch.cuda.is_available() else 0) < 2:
        assert bench.main(["--gpus", "2", *SMALL]) == 2
        assert "refusing" in capsys.readouterr().err
