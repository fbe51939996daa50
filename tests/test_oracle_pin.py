"""Pins the plain-C oracle restatement (oracle/lamm_oracle.c) to the reference.

1. against the committed golden vectors tests/golden/reference_v1.npz, written
   by the unmodified reference (tests/golden/make_golden.py) — runs anywhere;
2. against oracle/_ref (the reference compiled from /root/reference) on fresh
   randomized inputs — bit-for-bit;
3. the SPEC.md known-answer cases.
"""
import os

import numpy as np
import pytest

import cases

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_v1.npz"))
SMALL = (16, 2, 4, 5.0, 3)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        return a.shape == b.shape and np.array_equal(bits(a), bits(b))
    return np.array_equal(a, b)


def batch_from(prefix):
    keys = ("atom_ptr", "pos", "Z", "dataset_index", "energy_mask", "force_mask", "energy", "forces", "denoise")
    return {k: GOLD[prefix + k] for k in keys}


# ------------------------------------------------------------- golden pin
def test_golden_neighbor_lists(oracle_port):
    b = batch_from("nlbatch_")
    ap = b["atom_ptr"]
    for s in range(len(ap) - 1):
        got = oracle_port.neighbor_list(b["pos"][ap[s]:ap[s + 1]], b["Z"][ap[s]:ap[s + 1]], 5.0)
        for k, g in zip("ijdu", got):
            assert same(g, GOLD[f"nl{s}_{k}"]), f"sample {s} field {k}"


def test_golden_model(oracle_port):
    b = batch_from("mol_")
    p = GOLD["params"]
    assert same(oracle_port.init_params(SMALL, 7), p)
    e, f = oracle_port.forward(SMALL, p, b)
    assert same(e, GOLD["energy"]) and same(f, GOLD["forces"])
    bd, ge, gf = oracle_port.loss_grad(b, SMALL[4], e, f)
    assert same([bd["total"], bd["energy_term"], bd["force_term"]], GOLD["loss"])
    assert same(ge, GOLD["g_energy"]) and same(gf, GOLD["g_forces"])
    assert same(oracle_port.backward(SMALL, p, b, ge, gf), GOLD["grads"])


def test_golden_train_step(oracle_port):
    mb = batch_from("mix_")
    t = {k: GOLD["table_" + k] for k in ("rho", "rho_has", "mean", "std", "fstd", "has")}
    st = oracle_port.train_step(SMALL, 2, 3, mb, t, GOLD["params"], np.zeros_like(GOLD["params"]), seed=11, step=2,
                                clip=0.05)
    assert same([st["loss"], st["grad_norm"]], GOLD["step_loss"])
    assert same(st["grads"], GOLD["step_grads"])
    assert same(st["params"], GOLD["step_params"]) and same(st["rms_v"], GOLD["step_v"])


def test_golden_scheduler_and_streams(oracle_port):
    tr = oracle_port.make_trace("lognormal", 5000, 2, 2000, mode=20, sigma=1.0, seed=3)
    assert same(tr, GOLD["trace"])
    for mode in ("balanced", "greedy_only", "naive"):
        pl = oracle_port.plan(tr, 4, 2, 50, 9, mode)
        for k in ("sample", "worker", "atoms", "split", "chunk_rank", "worker_atoms"):
            assert same(pl[k], GOLD[f"plan_{mode}_{k}"]), (mode, k)
        stats = [pl["n_batches"], pl["dropped"], pl["max_imbalance"], pl["mean_imbalance"],
                 pl["monotonicity_violations"], pl["growth_events"]]
        assert same(np.array(stats, np.float64), GOLD[f"plan_{mode}_stats"]), mode
    assert same(oracle_port.rng_normals(123, 257), GOLD["normals"])
    assert same(oracle_port.rng_permutation(5, 100), GOLD["perm"])
    b = batch_from("mol_")
    x, lab = oracle_port.apply_noise(b["pos"][:5], b["Z"][:5], 0.3, 1, 99)
    assert same(x, GOLD["denoise_noisy"]) and same(lab, GOLD["denoise_labels"])


# --------------------------------------------------- randomized ref pin
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_equals_reference_model(oracle_port, oracle_ref, seed):
    cfg = cases.CFG
    b = cases.with_heads(cases.molecules(oracle_ref, 10, seed), cfg[4], seed)
    p = oracle_ref.init_params(cfg, seed)
    assert same(oracle_port.init_params(cfg, seed), p)
    e, f = oracle_ref.forward(cfg, p, b)
    e2, f2 = oracle_port.forward(cfg, p, b)
    assert same(e, e2) and same(f, f2)
    bd, ge, gf = oracle_ref.loss_grad(b, cfg[4], e, f)
    bd2, ge2, gf2 = oracle_port.loss_grad(b, cfg[4], e, f)
    assert bd == bd2 and same(ge, ge2) and same(gf, gf2)
    assert same(oracle_ref.backward(cfg, p, b, ge, gf), oracle_port.backward(cfg, p, b, ge, gf))
    ap = b["atom_ptr"]
    h, mt = oracle_ref.forward_cache(cfg, p, b["pos"][:ap[1]], b["Z"][:ap[1]])
    h2, mt2 = oracle_port.forward_cache(cfg, p, b["pos"][:ap[1]], b["Z"][:ap[1]])
    assert same(h, h2) and same(mt, mt2)


@pytest.mark.parametrize("G,B", [(1, 8), (2, 4), (4, 2)])
def test_port_equals_reference_train_step(oracle_port, oracle_ref, G, B):
    cfg = (32, 2, 8, 5.0, 4)
    b = cases.mixed_batch(oracle_ref, D=4, seed=G * 10 + B, count=G * B)
    t = cases.random_table(4, seed=G)
    p = oracle_ref.init_params(cfg, 3)
    v = np.full_like(p, 1e-4)
    r1 = oracle_ref.train_step(cfg, G, B, b, t, p, v, seed=5, step=7, clip=0.5)
    r2 = oracle_port.train_step(cfg, G, B, b, t, p, v, seed=5, step=7, clip=0.5)
    for k in ("params", "rms_v", "grads"):
        assert same(r1[k], r2[k]), k
    assert r1["loss"] == r2["loss"] and r1["grad_norm"] == r2["grad_norm"]


def test_port_equals_reference_scheduler(oracle_port, oracle_ref):
    tr = oracle_ref.make_trace("bimodal", 20000, 2, 2000, seed=8)
    assert same(tr, oracle_port.make_trace("bimodal", 20000, 2, 2000, seed=8))
    for mode in ("balanced", "greedy_only", "naive"):
        a, c = oracle_ref.plan(tr, 8, 4, 100, 2, mode), oracle_port.plan(tr, 8, 4, 100, 2, mode)
        for k in ("sample", "worker", "atoms", "split", "chunk_rank", "worker_atoms", "n_batches", "dropped",
                  "max_imbalance", "mean_imbalance", "monotonicity_violations", "growth_events"):
            assert same(a[k], c[k]), (mode, k)


def test_port_equals_reference_data(oracle_port, oracle_ref):
    kw = dict(mode=20, sigma=0.5, min_atoms=5, max_atoms=60, elements=cases.ORGANIC, offsets={1: -0.5, 8: 2.0})
    for task in ("energy_and_forces", "energy_only", "denoising"):
        a = oracle_ref.synth_generate(20, 4, task=task, **kw)
        c = oracle_port.synth_generate(20, 4, task=task, **kw)
        for k in a:
            assert same(a[k], c[k]), (task, k)
    sizes = [134e6, 8.2e6, 29e6, 9.5e6, 4.2e6, 2.0e6, 94e6, 460e3, 46e3, 132e3]
    assert same(oracle_ref.temperature_counts(sizes, 2.0), oracle_port.temperature_counts(sizes, 2.0))
    r = oracle_ref.temperature_counts([50, 20, 3], 2.0)
    a, c = oracle_ref.build_epoch_index(r, [50, 20, 3], 6), oracle_port.build_epoch_index(r, [50, 20, 3], 6)
    assert same(a[0], c[0]) and same(a[1], c[1])


# ------------------------------------------------------------- SPEC KATs
def test_spec_kat_neighbor_list(oracle_port):
    i, j, d, u = oracle_port.neighbor_list([[0, 0, 0], [1, 0, 0]], [1, 1], 5.0)
    assert len(i) == 2 and np.all(d == 1.0)
    assert len(oracle_port.neighbor_list([[0, 0, 0], [6, 0, 0]], [1, 1], 5.0)[0]) == 0
    rng = np.random.default_rng(1)
    pos = rng.uniform(0, 8, (10, 3))
    i, j, d, u = oracle_port.neighbor_list(pos, np.ones(10), 4.0)
    brute = [(a, b) for a in range(10) for b in range(10) if a != b and np.linalg.norm(pos[a] - pos[b]) < 4.0]
    assert list(zip(i.tolist(), j.tolist())) == brute
    assert np.all(np.abs(np.linalg.norm(u, axis=1) - 1) < 1e-12)


def test_spec_kat_loss(oracle_port):
    # B=1, N=2, energy error 0.5, per-atom force error norms 1 and 3 -> L = 0.5 + (1+3)/2 = 2.5
    b = dict(atom_ptr=np.array([0, 2]), dataset_index=np.zeros(1, np.int32), energy_mask=np.ones(1, np.uint8),
             force_mask=np.ones(1, np.uint8), energy=np.array([1.0]), forces=np.zeros((2, 3)))
    bd, _, _ = oracle_port.loss_grad(b, 1, np.array([[1.5]]), np.array([1.0, 0, 0, 0, 3.0, 0]))
    assert bd["total"] == 2.5


def test_spec_kat_denoise(oracle_port):
    x = np.zeros((2, 3))
    d = np.array([[1.0, 0, 0], [3.0, 0, 0]])
    noisy, lab = oracle_port.apply_displacements(x, [1, 1], d, 1)
    assert np.array_equal(lab, [[1, 0, 0], [-1, 0, 0]]) and np.array_equal(noisy, [[-1, 0, 0], [1, 0, 0]])
    _, lab = oracle_port.apply_displacements(x, [1, 1], d, 0)
    assert np.array_equal(lab, [[-1, 0, 0], [-3, 0, 0]])
    _, lab = oracle_port.apply_noise(np.zeros((1, 3)), [6], 0.3, 1, 4)
    assert not np.any(lab)


def test_spec_kat_greedy(oracle_port):
    assert oracle_port.greedy_assign([8, 7, 2, 1], 2, 2).tolist() == [0, 1, 1, 0]
    assert oracle_port.greedy_assign([5, 5, 5, 5], 2, 2).tolist() == [0, 1, 0, 1]
    assert oracle_port.greedy_assign([4, 9, 2], 1, 3).tolist() == [0, 0, 0]
