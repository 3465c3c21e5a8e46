"""The command-line front end (paper_2007_04457_b200/lib/hgr-b200), restating
the reference's tests/test_cli.sh: exit codes (0 ok, 1 usage, 2 data/format),
--json reports, deterministic .hg bytes (identical to the reference's
write_file), prefix-read byte accounting, f32 non-uniform round trip.
The header/usage/error subcommands run on the host; decompose/recompose need a GPU."""
import json
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2007_04457_b200" / "lib" / "hgr-b200"


def run(*args):
    if not CLI.exists():
        pytest.fail(f"{CLI} not built (make -C paper_2007_04457_b200/csrc)")
    p = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True)
    return p.returncode, p.stdout, p.stderr


def smooth(dims, dtype):
    # tests/gen_raw.cpp:46-47 ("smooth" pattern), row-major
    ext = list(dims) + [1] * (3 - len(dims))
    i, j, k = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in ext], indexing="ij")
    v = np.sin(0.21 * i) * np.cos(0.13 * j) + 0.5 * np.sin(0.07 * k)
    return v.reshape(dims).astype(dtype)


def test_usage_errors_exit_1():
    assert run()[0] == 1
    assert run("decompose", "--nope")[0] == 1
    assert run("bogus")[0] == 1
    assert run("decompose", "--input", "x", "--dims", "a,b", "--output", "y")[0] == 1


def test_info_and_error_on_host(tmp_path):
    if not oracle.available("reference"):
        pytest.skip("reference oracle not built")
    O = oracle.Oracle("reference")
    u = smooth((33, 33, 33), np.float64)
    p = O.decompose(u)
    f = tmp_path / "a.hg"
    nbytes = O.write_file(p, f)
    rc, out, err = run("info", "--input", f, "--json")
    assert rc == 0, err
    j = json.loads(out)
    assert out.count("\n") == 1 and j["classes"] == 6 and j["file_bytes"] == nbytes
    assert j["dims"] == [33, 33, 33] and j["precision_bytes"] == 8 and j["command"] == "info"
    assert list(j) == sorted(j)  # nlohmann::json key order
    rc, out, _ = run("info", "--input", f)
    assert rc == 0 and "6 classes" in out
    raw = tmp_path / "a.raw"
    u.tofile(raw)
    assert run("info", "--input", raw)[0] == 2  # garbage .hg -> data error
    noisy = tmp_path / "n.raw"
    (u + 1e-3).tofile(noisy)
    rc, out, _ = run("error", "--original", raw, "--reconstruction", noisy, "--precision", "f64",
                     "--json")
    assert rc == 0
    j = json.loads(out)
    assert abs(j["linf_abs"] - 1e-3) < 1e-12
    assert run("error", "--original", raw, "--reconstruction", f, "--precision", "f64")[0] == 2


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path, cuda):
    a = tmp_path / "a.raw"
    smooth((33, 33, 33), np.float64).tofile(a)
    rc, out, err = run("decompose", "--input", a, "--dims", "33,33,33", "--precision", "f64",
                       "--output", tmp_path / "a.hg")
    assert rc == 0, err
    assert "classes: 6" in out
    run("decompose", "--input", a, "--dims", "33,33,33", "--precision", "f64",
        "--output", tmp_path / "a2.hg")
    assert (tmp_path / "a.hg").read_bytes() == (tmp_path / "a2.hg").read_bytes()
    if oracle.available("reference"):
        O = oracle.Oracle("reference")
        O.write_file(O.decompose(np.fromfile(a).reshape(33, 33, 33)), tmp_path / "ref.hg")
        # the GPU decompose rounds differently (FMA contraction, K*P identity), so the
        # payloads agree to tolerance while the headers agree byte for byte
        ours, ref = (tmp_path / "a.hg").read_bytes(), (tmp_path / "ref.hg").read_bytes()
        assert len(ours) == len(ref)
        h = json.loads(run("info", "--input", tmp_path / "a.hg", "--json")[1])["header_bytes"]
        assert ours[:h] == ref[:h]
        x = np.frombuffer(ours[h:], np.float64)
        y = np.frombuffer(ref[h:], np.float64)
        assert np.abs(x - y).max() <= 1e-12 * 1.5
    rc, out, _ = run("info", "--input", tmp_path / "a.hg", "--json")
    file_bytes = json.loads(out)["file_bytes"]
    rc, out, err = run("recompose", "--input", tmp_path / "a.hg", "--classes", 5,
                       "--output", tmp_path / "r5.raw", "--json")
    assert rc == 0, err
    assert json.loads(out)["bytes_read"] == file_bytes
    rc, out, _ = run("error", "--original", a, "--reconstruction", tmp_path / "r5.raw",
                     "--precision", "f64", "--json")
    assert json.loads(out)["l2_rel"] <= 1e-12
    rc, out, _ = run("recompose", "--input", tmp_path / "a.hg", "--classes", 0,
                     "--output", tmp_path / "r0.raw", "--json")
    b0 = json.loads(out)["bytes_read"]
    assert b0 < file_bytes
    rc, out, _ = run("error", "--original", a, "--reconstruction", tmp_path / "r0.raw",
                     "--precision", "f64", "--json")
    assert 1e-12 < json.loads(out)["l2_rel"] < 1.5
    # a 513-node line refactors into ten classes
    line = tmp_path / "line.raw"
    smooth((513,), np.float64).tofile(line)
    rc, out, _ = run("decompose", "--input", line, "--dims", 513, "--precision", "f64",
                     "--uniform", "--output", tmp_path / "line.hg")
    assert rc == 0 and "classes: 10" in out
    # data errors exit 2
    rc, _, err = run("decompose", "--input", a, "--dims", "10,10", "--precision", "f64",
                     "--output", tmp_path / "x.hg")
    assert rc == 2 and "2^k+1" in err
    assert run("decompose", "--input", a, "--dims", "33,33", "--precision", "f64",
               "--output", tmp_path / "x.hg")[0] == 2
    assert run("decompose", "--input", tmp_path / "nothere.raw", "--dims", "33,33,33",
               "--precision", "f64", "--output", tmp_path / "x.hg")[0] == 2
    assert run("recompose", "--input", tmp_path / "a.hg", "--classes", 9,
               "--output", tmp_path / "x.raw")[0] == 2
    # non-uniform coordinates via per-dimension files, f32
    b = tmp_path / "b.raw"
    oracle.random_values(17 * 9, 12345).astype(np.float32).tofile(b)
    (tmp_path / "cx.txt").write_text("".join(f"{i}.5\n" for i in range(17)))
    (tmp_path / "cy.txt").write_text("".join(f"{i * i + i:.6f}\n" for i in range(9)))
    rc, _, err = run("decompose", "--input", b, "--dims", "17,9", "--precision", "f32",
                     "--coords-file", tmp_path / "cx.txt", "--coords-file", tmp_path / "cy.txt",
                     "--output", tmp_path / "b.hg")
    assert rc == 0, err
    assert run("recompose", "--input", tmp_path / "b.hg", "--classes", 3,
               "--output", tmp_path / "b3.raw")[0] == 0
    rc, out, _ = run("error", "--original", b, "--reconstruction", tmp_path / "b3.raw",
                     "--precision", "f32", "--json")
    assert json.loads(out)["l2_rel"] <= 1e-5


def test_rank_configs_matches_reference_model():
    """rank-configs (hgr_main.cpp:230-286): ranks and modeled seconds equal the
    reference's perf_model.hpp estimate_time; (2,2,2) ranks last (test_cli.sh:72-79)."""
    import ctypes as C
    rc, out, err = run("rank-configs", "--n", 513, "--bytes-per-element", 8, "--ghost", 4, "--json")
    assert rc == 0, err
    assert '"bx":2,"by":2,"bz":2,"rank":7' in out
    j = json.loads(out)
    assert list(j) == sorted(j) and j["n"] == 513
    if oracle.available("reference"):
        lib = C.CDLL(str(oracle.REF_SO))
        f = lib.hgrref_estimate_time
        f.restype = C.c_double
        f.argtypes = [C.c_int] + [C.c_ulonglong] * 7 + [C.c_double]
        for kind, name in enumerate(("GPK", "LPK", "IPK")):
            for e in j[name]:
                want = f(kind, e["bx"], e["by"], e["bz"], 513, 32, 8, 4, 1.0)
                assert e["seconds"] == want, (name, e)
    (Path(os.environ.get("TMPDIR", "/tmp")) / "hgr_cfgs.txt").write_text("8 4 4\n2,2,2\n# c\n16 4 4\n")
    rc, out, _ = run("rank-configs", "--configs",
                     Path(os.environ.get("TMPDIR", "/tmp")) / "hgr_cfgs.txt", "--kernel", "gpk",
                     "--top", 1)
    assert rc == 0 and "rank" in out
    assert run("rank-configs", "--top", 9)[0] == 2  # data error
    assert run("rank-configs", "--kernel", "xyz")[0] == 1  # usage error
