"""The C++ host side (include/cashash_b200/cashash.hpp): compiled with g++ against libchgpu.so and
the CPU oracle, then run.  The program's own checks mirror the reference library's call sequence
(build_hash_family -> set_centering -> compute_codes -> match_pair -> save_matches)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

import oracle_lib

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_1805_08995_b200"
EXE = ROOT / "tests" / "cpp" / "_build" / "facade_test"


def build_exe() -> Path:
    from paper_1805_08995_b200 import build as b

    b.build_all()
    oracle_lib.build_oracle(ref=False)
    src = ROOT / "tests" / "cpp" / "facade_test.cpp"
    hdr = ROOT / "include" / "cashash_b200" / "cashash.hpp"
    libs = [PKG / "libchgpu.so", ROOT / "oracle" / "libchoracle.so"]
    EXE.parent.mkdir(exist_ok=True)
    if not EXE.exists() or EXE.stat().st_mtime < max(p.stat().st_mtime for p in [src, hdr, *libs]):
        subprocess.run(["g++", "-std=gnu++20", "-O1", "-Wall", "-I", str(ROOT / "include"), "-I", str(ROOT / "oracle"),
                        str(src), "-o", str(EXE), f"-L{PKG}", f"-L{ROOT / 'oracle'}", "-lchgpu", "-lchoracle",
                        f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{ROOT / 'oracle'}"], check=True)
    return EXE


def run(*args):
    exe = build_exe()
    r = subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=600)
    sys.stdout.write(r.stdout)
    sys.stderr.write(r.stderr)
    assert r.returncode == 0, r.stderr
    assert "facade_test ok" in r.stdout


def test_facade_host_side():
    run("--host")


@pytest.mark.gpu
def test_facade_against_oracle_on_device():
    run()
