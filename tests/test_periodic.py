"""Periodic cells: image neighbour lists (minimum image for
cells at least 2 rc wide, every image within rc for narrower cells, per-axis
periodicity for slabs) and the model on periodic crystals. The reference has no
cells, so this extension is parity-unpinned against it: the checker is the
plain-C oracle (oracle/lamm_oracle.c:image_disp / build_pairs_cell), itself
checked here against an independent numpy image enumeration."""
import numpy as np
import pytest

import cases
from conftest import TOL, assert_close


def _image_pairs(pos, cell, rc):
    """All (i, j, r) with r < rc over the 27 neighbouring images (widths >= 2 rc:
    at most one image per pair)."""
    out = []
    shifts = np.array([[a, b, c] for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]) @ cell
    for i in range(len(pos)):
        for j in range(len(pos)):
            if i == j:
                continue
            d = pos[i] - pos[j] + shifts
            r = np.linalg.norm(d, axis=1)
            hit = np.nonzero(r < rc)[0]
            assert len(hit) <= 1
            if len(hit):
                out.append((i, j, r[hit[0]]))
    return out


def _all_images(pos, cell, rc, pbc=(1, 1, 1)):
    """Independent enumeration: {(i, j): sorted distances} over every image shift
    n (|n_k| <= ceil(rc / width_k) + 1 on periodic axes, 0 on open ones), n = 0
    excluded for i == j."""
    cell = np.asarray(cell, float)
    inv = np.linalg.inv(cell)
    M = [int(np.ceil(rc * np.linalg.norm(inv[:, k]))) + 1 if pbc[k] else 0 for k in range(3)]
    shifts = np.array([[a, b, c] for a in range(-M[0], M[0] + 1) for b in range(-M[1], M[1] + 1)
                       for c in range(-M[2], M[2] + 1)], float)
    out = {}
    for i in range(len(pos)):
        for j in range(len(pos)):
            d = pos[i] - pos[j] - shifts @ cell
            r = np.linalg.norm(d, axis=1)
            keep = r < rc
            if i == j:
                keep &= np.any(shifts != 0, axis=1)
            if keep.any():
                out[(i, j)] = np.sort(r[keep])
    return out


def image_cases():
    """(name, pos, Z, cell, pbc): cells narrower than 2 rc (several images per pair,
    self-images), a triclinic 2-atom cell, slabs (an open axis) and one large
    (> kSmallAtoms) sample that needs images."""
    rng = np.random.default_rng(7)
    out = []
    p, z, c = cases.diamond_supercell(reps=1, seed=1)                    # 8-atom Si cell, a = 5.43 A
    out.append(("si8", p, z, c, (1, 1, 1)))
    a = 5.43 / 2
    c2 = np.array([[0, a, a], [a, 0, a], [a, a, 0]], float)               # 2-atom primitive Si (triclinic)
    out.append(("si2", np.array([[0, 0, 0], [a / 2, a / 2, a / 2]]) + rng.normal(0, 0.02, (2, 3)),
                np.array([14, 14], np.int32), c2, (1, 1, 1)))
    out.append(("sc1", np.zeros((1, 3)), np.array([6], np.int32), np.eye(3) * 2.5, (1, 1, 1)))  # 1 atom, m = 2
    p, z, c = cases.diamond_supercell(reps=(2, 2, 1), seed=3)             # slab: open along the third vector
    c[2, 2] = 30.0
    out.append(("slab32", p, z, c, (1, 1, 0)))
    p, z, c = cases.diamond_supercell(reps=(2, 1, 3), seed=4)             # mixed widths 10.86 / 5.43 / 16.3
    out.append(("mixed48", p, z, c, (1, 1, 1)))
    p, z, c = cases.diamond_supercell(reps=(5, 5, 1), seed=5)             # 200 atoms, 5.43 A along c: images
    out.append(("wide200", p, z, c, (1, 1, 1)))
    return out


@pytest.mark.parametrize("case", image_cases(), ids=lambda c: c[0])
def test_oracle_images_vs_enumeration(oracle_port, case):
    name, pos, Z, cell, pbc = case
    with oracle_port.periodic(cell[None], pbc=np.array([pbc], np.uint8)):
        i, j, dist, unit = oracle_port.neighbor_list(pos, Z, 5.0)
    ref = _all_images(pos, cell, 5.0, pbc)
    got = {}
    for a, b, r in zip(i.tolist(), j.tolist(), dist.tolist()):
        got.setdefault((a, b), []).append(r)
    assert sorted(got) == sorted(ref), name
    for k, v in ref.items():
        assert np.allclose(np.sort(got[k]), v, rtol=0, atol=1e-12), (name, k)
    # order: i-major, j ascending (images of one (i, j) contiguous)
    key = i.astype(np.int64) * (len(pos) + 1) + j
    assert np.all(np.diff(key) >= 0), name
    assert np.allclose(np.linalg.norm(unit, axis=1), 1.0, atol=1e-12)
    if name == "si8":  # bulk Si: the same 28 neighbours per atom as the supercells
        assert len(i) == 8 * 28
    if name == "sc1":  # simple cubic 2.5 A: 6 + 12 + 8 + 6 + 24 (r = 2.5, 3.54, 4.33, 5.0 excluded, 5.59 out)
        assert len(i) == 6 + 12 + 8


def test_cell_inverse_same_bits_in_product_and_oracle(oracle_port):
    import paper_2505_22208_b200 as pk
    rng = np.random.default_rng(0)
    for _ in range(50):
        cell = np.eye(3) * rng.uniform(8, 20) + rng.normal(0, 2, (3, 3))
        assert np.array_equal(pk.cell_inverse(cell).view(np.uint64), oracle_port.cell_inverse(cell).view(np.uint64))


@pytest.mark.parametrize("which", ["diamond", "triclinic"])
def test_oracle_minimum_image_vs_image_enumeration(oracle_port, which):
    pos, Z, cell = cases.diamond_supercell(seed=1) if which == "diamond" else cases.triclinic_box(seed=2)
    with oracle_port.periodic(cell[None]):
        i, j, dist, unit = oracle_port.neighbor_list(pos, Z, 5.0)
    ref = _image_pairs(pos, cell, 5.0)
    assert [(a, b) for a, b, _ in ref] == list(zip(i.tolist(), j.tolist()))
    assert np.allclose(dist, [r for _, _, r in ref], rtol=0, atol=1e-12)
    assert np.allclose(np.linalg.norm(unit, axis=1), 1.0, atol=1e-12)
    if which == "diamond":  # shells within 5 A: 4 at a sqrt(3)/4, 12 at a/sqrt(2), 12 at a sqrt(11)/4
        assert len(i) == len(pos) * 28


@pytest.mark.gpu
def test_periodic_neighbor_list_bit_exact(pk, dev, oracle_port):
    b = cases.periodic_batch(pk)
    dev.set_batch(b)
    ptr, gi, gj, gd, gu = dev.build_neighbor_list(fp64=True)
    ap = b["atom_ptr"]
    for s in range(len(ap) - 1):
        cell = np.asarray(b["cell"][s])
        with oracle_port.periodic(cell[None]):
            i, j, dist, unit = oracle_port.neighbor_list(b["pos"][ap[s]:ap[s + 1]], b["Z"][ap[s]:ap[s + 1]], 5.0)
        lo, hi = ptr[s], ptr[s + 1]
        assert np.array_equal(gi[lo:hi], i) and np.array_equal(gj[lo:hi], j), s
        assert np.array_equal(gd[lo:hi].view(np.uint64), dist.view(np.uint64)), s
        assert np.array_equal(gu[lo:hi].view(np.uint64), unit.view(np.uint64)), s


@pytest.mark.gpu
def test_periodic_cell_list_bit_exact(pk, dev, oracle_port):
    """Periodic samples above kSmallAtoms: 3, 4 and 5 slabs per lattice direction
    (diamond supercells) and 2 (a skewed cell just over 2 rc wide, where the -1 and
    +1 neighbour slabs are the same one)."""
    parts = []
    for reps in (3, 4, 5):
        pos, Z, cell = cases.diamond_supercell(reps=reps, seed=reps)
        parts.append((pos, Z, cell))
    parts.append(cases.triclinic_box(n=150, seed=4, cell=((12.0, 0.0, 0.0), (1.0, 11.5, 0.0), (0.5, 1.0, 11.2))))
    b = pk.concat([dict(cases.pack([(p, z)]), cell=c[None]) for p, z, c in parts] + [cases.molecules(pk, 3, 2)])
    dev.set_batch(b)
    ptr, gi, gj, gd, gu = dev.build_neighbor_list(fp64=True)
    ap = b["atom_ptr"]
    for s in range(len(parts)):
        cell = np.asarray(b["cell"][s])
        with oracle_port.periodic(cell[None]):
            i, j, dist, unit = oracle_port.neighbor_list(b["pos"][ap[s]:ap[s + 1]], b["Z"][ap[s]:ap[s + 1]], 5.0)
        lo, hi = ptr[s], ptr[s + 1]
        assert np.array_equal(gi[lo:hi], i) and np.array_equal(gj[lo:hi], j), s
        assert np.array_equal(gd[lo:hi].view(np.uint64), dist.view(np.uint64)), s
        assert np.array_equal(gu[lo:hi].view(np.uint64), unit.view(np.uint64)), s
    assert ptr[1] - ptr[0] == 216 * 28


@pytest.mark.gpu
@pytest.mark.parametrize("large", [False, True])
def test_periodic_train_step_matches_oracle(pk, oracle_port, large):
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    b = cases.periodic_batch(pk, seed=5, large=large)
    B = len(b["atom_ptr"]) - 1
    table = cases.random_table(cases.CFG[4], seed=4)
    params = oracle_port.init_params(cases.CFG, 8)
    tc = pk.TrainConfig(seed=2, clip_norm=1e9)
    with oracle_port.periodic(b["cell"]):
        ref = oracle_port.train_step(cases.CFG, 1, B, b, table, params, np.zeros_like(params), seed=2, step=0,
                                     clip=1e9)
        re, rf = oracle_port.forward(cases.CFG, params, b)
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_rms_state(np.zeros_like(params))
    dev.set_reference_table(None)
    dev.set_batch(b)
    e, f = dev.forward()
    assert_close(e, re, what="periodic energies")
    assert_close(f, rf, what="periodic forces")
    dev.set_reference_table(table)
    res = dev.train_step(b, tc, step=0)
    assert abs(res.loss - ref["loss"]) <= TOL * abs(ref["loss"])
    assert_close(dev.grads(), ref["grads"], what="periodic gradient")
    dev.close()


def image_batch(pk, seed=11, D=10):
    """Every image case plus a minimum-image crystal and molecules in one batch."""
    rng = np.random.default_rng(seed)
    parts = []
    for name, pos, Z, cell, pbc in image_cases():
        n = len(Z)
        parts.append(dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z, forces=rng.normal(0, 1, (n, 3)),
                          dataset_index=np.zeros(1, np.int32), energy_mask=np.ones(1, np.uint8),
                          force_mask=np.ones(1, np.uint8), energy=rng.normal(-3.0 * n, 1.0, 1),
                          denoise=np.zeros(1, np.uint8), cell=cell[None], pbc=np.array([pbc], np.uint8)))
    b = pk.concat(parts + [cases.periodic_batch(pk, D=D, seed=seed)])
    b["dataset_index"] = rng.integers(0, D, len(b["atom_ptr"]) - 1).astype(np.int32)
    return b


@pytest.mark.gpu
def test_image_neighbor_lists_bit_exact(pk, dev, oracle_port):
    """Narrow cells, slabs and a large sample that needs images, next to minimum-image
    crystals and molecules: pairs, order, fp64 distances and unit vectors bit-exact."""
    b = image_batch(pk)
    dev.set_batch(b)
    ptr, gi, gj, gd, gu = dev.build_neighbor_list(fp64=True)
    ap = b["atom_ptr"]
    for s in range(len(ap) - 1):
        cell = np.asarray(b["cell"][s])
        with oracle_port.periodic(cell[None], pbc=b["pbc"][s][None]):
            i, j, dist, unit = oracle_port.neighbor_list(b["pos"][ap[s]:ap[s + 1]], b["Z"][ap[s]:ap[s + 1]], 5.0)
        lo, hi = ptr[s], ptr[s + 1]
        assert np.array_equal(gi[lo:hi], i) and np.array_equal(gj[lo:hi], j), s
        assert np.array_equal(gd[lo:hi].view(np.uint64), dist.view(np.uint64)), s
        assert np.array_equal(gu[lo:hi].view(np.uint64), unit.view(np.uint64)), s


@pytest.mark.gpu
def test_image_train_step_matches_oracle(pk, oracle_port):
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    b = image_batch(pk, seed=12)
    B = len(b["atom_ptr"]) - 1
    b["denoise"][::3] = 1
    table = cases.random_table(cases.CFG[4], seed=4, elements=(1, 6, 7, 8, 14))
    params = oracle_port.init_params(cases.CFG, 8)
    tc = pk.TrainConfig(seed=2, clip_norm=1e9)
    with oracle_port.periodic(b["cell"], pbc=b["pbc"]):
        ref = oracle_port.train_step(cases.CFG, 1, B, b, table, params, np.zeros_like(params), seed=2, step=0,
                                     clip=1e9)
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_rms_state(np.zeros_like(params))
    dev.set_reference_table(table)
    res = dev.train_step(b, tc, step=0)
    assert abs(res.loss - ref["loss"]) <= TOL * abs(ref["loss"])
    assert_close(dev.grads(), ref["grads"], what="image-cell gradient")
    dev.close()


@pytest.mark.gpu
def test_periodic_cell_far_too_small_is_input_error(pk, dev):
    """A 0.3 A cell needs 35^3 images per pair (> 4096): LAMM_EINPUT."""
    b = dict(atom_ptr=np.array([0, 1], np.int64), pos=np.zeros((1, 3)), Z=np.array([6], np.int32),
             cell=(np.eye(3) * 0.3)[None])
    with pytest.raises(pk.InputError):
        dev.set_batch(b)
