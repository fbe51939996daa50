"""Periodic cells: minimum-image neighbour lists and the
model on periodic crystals. The reference has no cells, so this extension is
parity-unpinned against it: the checker is the plain-C oracle's minimum image
(oracle/lamm_oracle.c:min_image), itself checked here against an independent
image enumeration."""
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


@pytest.mark.gpu
def test_periodic_cell_too_small_is_input_error(pk, dev):
    pos, Z, cell = cases.diamond_supercell(reps=1)  # 5.43 A < 2 * cutoff
    b = dict(atom_ptr=np.array([0, len(Z)], np.int64), pos=pos, Z=Z, cell=cell[None])
    with pytest.raises(pk.InputError):
        dev.set_batch(b)
