"""Seeded inputs shared by the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

CFG = (128, 3, 16, 5.0, 10)  # LaMM-sized ModelConfig{hidden, layers, rbf, cutoff, heads}
ORGANIC = (1, 6, 7, 8)


def synth(lib, count, seed, **kw):
    """Reference generator (S/dataset.cpp:234-247) through any binding."""
    return lib.synth_generate(count, seed, **kw)


def molecules(lib, count=32, seed=42):
    """cfg2-like: lognormal(mode 20, sigma 0.5) molecules, 5-60 atoms, elements {1,6,7,8}."""
    return synth(lib, count, seed, mode=20, sigma=0.5, min_atoms=5, max_atoms=60, elements=ORGANIC)


def with_heads(batch, D, seed=0):
    """Assigns dataset indices (heads) pseudo-randomly in [0, D)."""
    b = dict(batch)
    b["dataset_index"] = np.random.default_rng(seed).integers(0, D, len(b["atom_ptr"]) - 1).astype(np.int32)
    return b


def pack(systems):
    """systems: list of (pos[n,3], Z[n]) -> unlabeled batch dict."""
    sizes = [len(z) for _, z in systems]
    ap = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    B, N = len(systems), int(ap[-1])
    return dict(atom_ptr=ap, pos=np.concatenate([np.asarray(p, float).reshape(-1, 3) for p, _ in systems]),
                Z=np.concatenate([np.asarray(z, np.int32) for _, z in systems]), dataset_index=np.zeros(B, np.int32),
                energy_mask=np.zeros(B, np.uint8), force_mask=np.zeros(B, np.uint8), energy=np.zeros(B),
                forces=np.zeros((N, 3)), denoise=np.zeros(B, np.uint8))


def edge_systems(rng):
    """SPEC.md:53-55 known answers plus boundary cases of the strict r < cutoff test."""
    s = []
    s.append((np.zeros((1, 3)), [6]))                                     # isolated atom: no pairs
    s.append(([[0, 0, 0], [1, 0, 0]], [1, 8]))                            # 1 A apart: 2 pairs, d = 1
    s.append(([[0, 0, 0], [6, 0, 0]], [6, 6]))                            # 6 A apart: 0 pairs
    s.append(([[0, 0, 0], [5, 0, 0]], [6, 7]))                            # exactly the cutoff: excluded
    s.append(([[0, 0, 0], [np.nextafter(5.0, 0.0), 0, 0]], [6, 7]))      # just inside
    s.append(([[0, 0, 0], [3, 4, 0], [0, 0, 5]], [1, 1, 1]))              # 3-4-5: r = 5 exactly, twice
    s.append((rng.uniform(0, 8, (10, 3)), rng.choice(ORGANIC, 10)))       # SPEC: 10 atoms in an 8 A box
    s.append((rng.uniform(-1, 1, (40, 3)) * 3.0, rng.choice(ORGANIC, 40)))  # dense, many pairs
    return s


def random_table(D, seed=0, elements=ORGANIC):
    """A ReferenceTable with reference energies for some elements (H/loss.hpp:31-44)."""
    rng = np.random.default_rng(seed)
    rho = np.zeros((D, 119))
    has = np.zeros((D, 119), np.uint8)
    for d in range(D):
        for z in elements:
            if rng.random() < 0.75:
                rho[d, z] = rng.normal(-2.0, 1.0)
                has[d, z] = 1
    return dict(rho=rho, rho_has=has, mean=rng.normal(0, 1, D), std=rng.uniform(0.5, 2.0, D),
                fstd=rng.uniform(0.5, 2.0, D), has=np.ones(D, np.uint8))


def mixed_batch(lib, D=10, seed=5, count=24, denoise_frac=0.3):
    """LaMM semi-supervised mix: E+F, E-only and denoising samples on several heads."""
    b = synth(lib, count, seed, mode=15, sigma=0.45, min_atoms=4, max_atoms=40, elements=ORGANIC)
    rng = np.random.default_rng(seed)
    B = count
    kind = rng.choice(3, B, p=[0.5, 0.2, 0.3]) if denoise_frac else np.zeros(B, int)
    b["dataset_index"] = rng.integers(0, D, B).astype(np.int32)
    b["force_mask"] = (kind == 0).astype(np.uint8)
    b["energy_mask"] = (kind != 2).astype(np.uint8)
    b["denoise"] = (kind == 2).astype(np.uint8)
    return b


def diamond_supercell(reps=2, a=5.43, jitter=0.05, seed=0, Z=14):
    """cfg1's periodic bulk: an reps^3 (or r0 x r1 x r2) diamond supercell (8 atoms
    per cubic cell, a = 5.43 A for Si) with Gaussian jitter; returns (pos [n,3],
    Z [n], cell [3,3])."""
    rng = np.random.default_rng(seed)
    r = np.broadcast_to(np.asarray(reps, int), (3,))
    basis = np.array([[0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0],
                      [.25, .25, .25], [.25, .75, .75], [.75, .25, .75], [.75, .75, .25]])
    frac = np.array([b + np.array([i, j, k]) for i in range(r[0]) for j in range(r[1]) for k in range(r[2])
                     for b in basis]) / r
    cell = np.diag(a * r.astype(float))
    pos = frac @ cell + rng.normal(0.0, jitter, (len(frac), 3))
    return pos, np.full(len(frac), Z, np.int32), cell


def triclinic_box(n=48, seed=0, cell=((11.5, 0.0, 0.0), (2.0, 11.0, 0.0), (1.0, 1.5, 10.8))):
    """Random atoms (rejection: > 1.3 A apart under the minimum image) in a skewed
    cell whose perpendicular widths exceed 2 * 5 A."""
    rng = np.random.default_rng(seed)
    cell = np.asarray(cell, np.float64)
    inv = np.linalg.inv(cell)
    pts = []
    while len(pts) < n:
        p = rng.uniform(0, 1, 3) @ cell
        ok = True
        for q in pts:
            d = p - q
            f = d @ inv
            d = (f - np.rint(f)) @ cell
            if np.linalg.norm(d) < 1.3:
                ok = False
                break
        if ok:
            pts.append(p)
    return np.array(pts), rng.choice(ORGANIC, n).astype(np.int32), cell


def periodic_batch(lib, D=10, seed=3, large=False):
    """A mixed batch: two periodic crystals (diamond Si supercell, triclinic box) and
    non-periodic molecules; labels from random values (parity only needs them finite).
    large: a 3x3x3 supercell (216 atoms) and a 150-atom triclinic box, i.e. samples
    above kSmallAtoms that take the cell-list path."""
    mol = molecules(lib, 6, seed)
    p1, z1, c1 = diamond_supercell(reps=3 if large else 2, seed=seed)
    p2, z2, c2 = triclinic_box(n=150 if large else 48, seed=seed + 1)
    rng = np.random.default_rng(seed)
    extra = []
    for p, z in ((p1, z1), (p2, z2)):
        n = len(z)
        extra.append(dict(atom_ptr=np.array([0, n], np.int64), pos=p, Z=z, forces=rng.normal(0, 1, (n, 3)),
                          dataset_index=np.zeros(1, np.int32), energy_mask=np.ones(1, np.uint8),
                          force_mask=np.ones(1, np.uint8), energy=rng.normal(-3.0 * n, 1.0, 1),
                          denoise=np.zeros(1, np.uint8), cell=None))
    extra[0]["cell"] = c1[None]
    extra[1]["cell"] = c2[None]
    mol = dict(mol)
    mol["denoise"] = np.zeros(len(mol["atom_ptr"]) - 1, np.uint8)
    b = lib_concat([extra[0], mol, extra[1]])
    b["dataset_index"] = rng.integers(0, D, len(b["atom_ptr"]) - 1).astype(np.int32)
    return b


def lib_concat(batches):
    import paper_2505_22208_b200 as pk
    return pk.concat(batches)
