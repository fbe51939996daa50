"""On-disk formats against the reference's own writers and
readers, compiled in oracle/_ref: LAMMCKPT checkpoints byte-identical both ways,
LAMMDS1 catalogs read into packed batches equal to read_catalog's samples."""
import os

import numpy as np
import pytest

import cases


@pytest.fixture(scope="module")
def io():
    from paper_2505_22208_b200 import io
    return io


def test_checkpoint_byte_identical_with_reference(tmp_path, io, oracle_ref):
    import paper_2505_22208_b200 as pk
    cfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    params = oracle_ref.init_params(cases.CFG, 5)
    ours, theirs = str(tmp_path / "ours.ckpt"), str(tmp_path / "ref.ckpt")
    io.save_checkpoint(ours, cfg, params)
    oracle_ref.checkpoint_save(theirs, cases.CFG, params)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    c2, p2 = io.load_checkpoint(theirs)  # ours reads theirs
    assert c2 == cfg and np.array_equal(p2.view(np.uint64), params.view(np.uint64))
    c3, p3 = oracle_ref.checkpoint_load(ours)  # theirs reads ours
    assert c3 == cases.CFG and np.array_equal(p3.view(np.uint64), params.view(np.uint64))


def test_checkpoint_errors(tmp_path, io):
    import paper_2505_22208_b200 as pk
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"NOTACKPT" + b"\\0" * 64)
    with pytest.raises(pk.InputError):
        io.load_checkpoint(str(bad))
    with pytest.raises(pk.InputError):
        io.load_checkpoint(str(tmp_path / "missing.ckpt"))


def test_rms_state_round_trip(tmp_path, io):
    import paper_2505_22208_b200 as pk
    cfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    v = np.random.default_rng(0).uniform(0, 1e-3, pk.param_count(cfg))
    io.save_rms_state(str(tmp_path / "v.rms"), cfg, v)
    c, v2 = io.load_rms_state(str(tmp_path / "v.rms"))
    assert c == cfg and np.array_equal(v.view(np.uint64), v2.view(np.uint64))


def test_catalog_reader_matches_reference(tmp_path, io, oracle_ref):
    d = str(tmp_path / "cat")
    oracle_ref.write_demo_catalog(d, 12, 9)
    ref, sizes = oracle_ref.read_catalog(d)
    cat = io.read_catalog(d)
    assert [len(s["batch"]["atom_ptr"]) - 1 for s in cat["subsets"]] == sizes.tolist()
    import paper_2505_22208_b200 as pk
    ours = pk.concat([s["batch"] for s in cat["subsets"]])
    for k in ("atom_ptr", "Z", "energy_mask", "force_mask", "dataset_index"):
        assert np.array_equal(ours[k], ref[k]), k
    for k in ("pos", "energy", "forces"):
        assert np.array_equal(ours[k].view(np.uint64), ref[k].view(np.uint64)), k
    assert [s["task"] for s in cat["subsets"]] == ["energy_and_forces", "energy_only", "denoising"]
    assert cat["subsets"][2]["batch"]["denoise"].all()


def test_subset_truncated_and_capacity(tmp_path, io, oracle_ref):
    """A truncated LAMMDS1 file fails in info (not a silent short count), and read
    refuses arrays smaller than the file declares."""
    import ctypes as C
    import paper_2505_22208_b200 as pk
    from paper_2505_22208_b200._lib import lib
    d = str(tmp_path / "cat")
    oracle_ref.write_demo_catalog(d, 6, 3)
    f = sorted(x for x in os.listdir(d) if x.endswith(".bin"))[0]
    path = os.path.join(d, f)
    full = open(path, "rb").read()
    b = io.read_subset(path)
    trunc = str(tmp_path / "trunc.bin")
    open(trunc, "wb").write(full[:-5])
    with pytest.raises(pk.InputError):
        io.read_subset(trunc)
    B, N = len(b["atom_ptr"]) - 1, int(b["atom_ptr"][-1])
    ap, pos, Z = np.empty(B + 1, np.int64), np.empty(3 * N), np.empty(N, np.int32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    for scap, acap in ((B - 1, N), (B, N - 1)):
        st = lib().lamm_subset_read(os.fsencode(path), 0, C.c_int64(scap), C.c_int64(acap), p(ap), p(pos), p(Z),
                                    None, None, None, None, None)
        assert st == 1
