"""The C++ drop-in header (include/hgr_b200/hgr.hpp) compiles like the
reference's headers and, on a GPU, passes the reference's known answers."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIBDIR = ROOT / "paper_2007_04457_b200" / "lib"


def _build(tmp_path):
    exe = tmp_path / "dropin_kat"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/dropin_kat.cpp"),
           f"-L{LIBDIR}", "-lhgr_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_dropin_known_answers(tmp_path, cuda):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
