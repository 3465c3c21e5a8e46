"""The .hg progressive container (storage.hpp:17-218), restating the reference's
test_storage.cpp cases. CPU tests: the header parser (hgr_hg_read_info, host-only
code of libhgr_b200.so) against files written by the reference itself
(oracle/_ref). GPU tests: files written from a device pyramid are
byte-identical to the reference's, and prefix reads scatter exactly the
reference's zero-filled pyramid."""
import os

import numpy as np
import pytest

import oracle


def _hgr():
    import paper_2007_04457_b200 as hgr
    return hgr


@pytest.fixture(scope="module")
def refo():
    if not oracle.available("reference"):
        pytest.skip("reference oracle (oracle/_ref) not built here")
    return oracle.Oracle("reference")


def sample(refo, shape, seed, dtype=np.float64, coords=None):
    u = oracle.random_values(int(np.prod(shape)), seed).reshape(shape).astype(dtype)
    return refo.decompose(u, coords)


# ---- CPU: header parsing of reference-written files ------------------------------

def test_five_node_layout_accounting(refo, tmp_path):
    hgr = _hgr()
    p = sample(refo, (5,), 3201)
    f = tmp_path / "c.hg"
    total = refo.write_file(p, f)
    info = hgr.read_info(f)
    assert info.class_count() == 3
    assert [info.class_elements(c) for c in range(3)] == [2, 1, 2]
    assert total - info.header_bytes == 40
    assert info.precision_bytes == 8 and info.extents == [5] and info.version == 1
    assert info.file_bytes == total == os.path.getsize(f)


def test_info_fields_nonuniform(refo, tmp_path):
    hgr = _hgr()
    coords = [oracle.random_coords(9, 3001), oracle.random_coords(17, 3002)]
    p = sample(refo, (9, 17), 3003, coords=coords)
    f = tmp_path / "a.hg"
    refo.write_file(p, f, coords)
    info = hgr.read_info(f)
    assert info.rank == 2 and info.extents == [9, 17]
    assert np.array_equal(info.coords[0], coords[0]) and np.array_equal(info.coords[1], coords[1])
    assert info.total_elements() == 9 * 17
    assert info.class_offsets[0] == info.header_bytes


def test_info_reads_the_header_only(refo, tmp_path):
    hgr = _hgr()
    p = sample(refo, (33,), 3401)
    f = tmp_path / "e.hg"
    refo.write_file(p, f)
    full = hgr.read_info(f)
    os.truncate(f, full.header_bytes + 8)
    info = hgr.read_info(f)
    assert info.class_count() == 6 and info.total_elements() == 33


def test_malformed_files_rejected(refo, tmp_path):
    hgr = _hgr()
    (tmp_path / "garbage.hg").write_bytes(b"this is not a refactored array")
    with pytest.raises(hgr.HgrError, match="magic"):
        hgr.read_info(tmp_path / "garbage.hg")
    (tmp_path / "empty.hg").write_bytes(b"")
    with pytest.raises(hgr.HgrError):
        hgr.read_info(tmp_path / "empty.hg")
    with pytest.raises(hgr.HgrError, match="cannot open"):
        hgr.read_info(tmp_path / "missing.hg")
    p = sample(refo, (5,), 3501)
    refo.write_file(p, tmp_path / "ok.hg")
    b = bytearray((tmp_path / "ok.hg").read_bytes())
    b[4] = 9
    (tmp_path / "badver.hg").write_bytes(bytes(b))
    with pytest.raises(hgr.HgrError, match="version"):
        hgr.read_info(tmp_path / "badver.hg")
    b = bytearray((tmp_path / "ok.hg").read_bytes())
    b[6] = 3  # precision code
    (tmp_path / "badprec.hg").write_bytes(bytes(b))
    with pytest.raises(hgr.HgrError, match="precision"):
        hgr.read_info(tmp_path / "badprec.hg")


# ---- GPU: write and prefix reads on the device ------------------------------------

CASES = [
    ((9, 17), np.float64, True, 3003),
    ((5, 9, 5), np.float32, False, 3004),
    ((9, 9), np.float64, False, 3101),
    ((5,), np.float64, False, 3201),
    ((17, 9), np.float64, False, 3301),
    ((33,), np.float64, False, 3401),
    ((65, 33, 129), np.float32, True, 3601),
    ((129, 65, 65), np.float64, False, 3602),
]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,dt,nonuniform,seed", CASES,
                         ids=lambda v: "x".join(map(str, v)) if isinstance(v, tuple) else str(v))
def test_write_matches_reference_bytes_and_prefix_reads(refo, cuda, tmp_path, shape, dt,
                                                        nonuniform, seed):
    import torch
    hgr = _hgr()
    coords = ([oracle.random_coords(n, seed + 11 * d) for d, n in enumerate(shape)]
              if nonuniform else None)
    p = sample(refo, shape, seed, dt, coords)
    g = hgr.GridHierarchy(coords) if coords else hgr.GridHierarchy.uniform(list(shape))
    ref_f, ours_f, again_f = tmp_path / "ref.hg", tmp_path / "ours.hg", tmp_path / "again.hg"
    nref = refo.write_file(p, ref_f, coords)
    r = hgr.RefactoredArray(torch.from_numpy(p).to(cuda), g)
    nours = hgr.write_file(r, ours_f)
    assert nours == nref == os.path.getsize(ours_f)
    assert ours_f.read_bytes() == ref_f.read_bytes()
    hgr.write_file(r, again_f)
    assert again_f.read_bytes() == ours_f.read_bytes()  # deterministic
    L = g.levels()
    full = hgr.read_prefix(ours_f, L)
    assert full.bytes_read == nref
    assert np.array_equal(full.array.data.cpu().numpy(), p)
    for m in range(L + 1):
        want, nbytes = refo.read_prefix(ref_f, m, shape, dt)
        got = hgr.read_prefix(ours_f, m)
        assert got.bytes_read == nbytes
        assert np.array_equal(got.array.data.cpu().numpy(), want), m
        # reconstruction from the prefix equals reconstruction from the full file
        a = hgr.recompose(got.array, m)
        b = hgr.recompose(full.array, m)
        assert torch.equal(a, b), m


@pytest.mark.gpu
def test_prefix_read_errors(refo, cuda, tmp_path):
    hgr = _hgr()
    p = sample(refo, (5,), 3501)
    f = tmp_path / "ok.hg"
    refo.write_file(p, f)
    for bad in (3, -1):
        with pytest.raises(hgr.HgrError, match="class index out of range"):
            hgr.read_prefix(f, bad)
    with pytest.raises(hgr.HgrError, match="precision"):
        hgr.read_prefix(f, 0, dtype="f32")
    q = sample(refo, (33,), 3401)
    t = tmp_path / "e.hg"
    refo.write_file(q, t)
    info = hgr.read_info(t)
    os.truncate(t, info.header_bytes + 8)
    with pytest.raises(hgr.HgrError, match="truncated"):
        hgr.read_prefix(t, info.class_count() - 1)
