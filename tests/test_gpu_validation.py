"""GPU edge cases of the train step: input validation (the reference's
`AtomicSystem::validate`, S/core.cpp:10-28, and the masked loss's dataset-index
check, S/loss.cpp:140-160) and batches the model must handle without edges or
without labels (an empty mask sum is a zero term plus a flag, S/loss.cpp:190-212).

Every invalid batch raises InputError (status 1) before anything is launched and
leaves the context usable: the next valid step is bit-identical to a fresh
context's. Edge-less and label-less batches match the reference step.
"""
import numpy as np
import pytest

from conftest import TOL, assert_close, has_gpu
import cases

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _mcfg(pk):
    return pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])


def _valid(pk):
    return cases.mixed_batch(pk, D=cases.CFG[4], seed=11, count=6, denoise_frac=0)


def _variant(b, **kw):
    out = {k: np.array(v, copy=True) for k, v in b.items()}
    out.update(kw)
    return out


def test_invalid_batches_raise_input_error_and_leave_the_context_usable(pk, oracle_ref):
    good = _valid(pk)
    B, N = len(good["atom_ptr"]) - 1, int(good["atom_ptr"][-1])
    params = oracle_ref.init_params(cases.CFG, 3)
    tc = pk.TrainConfig(seed=5, clip_norm=1e9)
    bad = {}
    ap = good["atom_ptr"].copy()
    ap[2] = ap[1]  # sample 1 empty (sample 2 starts where it did)
    bad["system without atoms"] = _variant(good, atom_ptr=ap)
    z = good["Z"].copy()
    z[3] = 0
    bad["Z = 0"] = _variant(good, Z=z)
    z = good["Z"].copy()
    z[N - 1] = 119
    bad["Z = 119"] = _variant(good, Z=z)
    p = good["pos"].copy()
    p[5, 1] = np.nan
    bad["NaN coordinate"] = _variant(good, pos=p)
    p = good["pos"].copy()
    p[0, 2] = np.inf
    bad["infinite coordinate"] = _variant(good, pos=p)
    ds = good["dataset_index"].copy()
    ds[B - 1] = cases.CFG[4]
    bad["dataset index = heads"] = _variant(good, dataset_index=ds)
    ds = good["dataset_index"].copy()
    ds[0] = -1
    bad["negative dataset index"] = _variant(good, dataset_index=ds)

    dev = pk.Device(_mcfg(pk), seed=0)
    dev.set_params(params)
    dev.set_rms_state(np.zeros_like(params))
    for what, b in bad.items():
        with pytest.raises(pk.InputError):
            dev.train_step(b, tc, step=1)
        with pytest.raises(pk.InputError):
            dev.stage(b, tc, step=1, slot=0)
    r = dev.train_step(good, tc, step=1)
    g = dev.grads()
    p1 = dev.params()
    dev.close()

    fresh = pk.Device(_mcfg(pk), seed=0)
    fresh.set_params(params)
    fresh.set_rms_state(np.zeros_like(params))
    r0 = fresh.train_step(good, tc, step=1)
    assert r.loss == r0.loss and r.grad_norm == r0.grad_norm
    assert np.array_equal(g, fresh.grads()) and np.array_equal(p1, fresh.params())
    fresh.close()


def test_edgeless_batch_matches_reference(pk, oracle_ref):
    """Isolated atoms and pairs beyond the cutoff: P = 0, every atom walks an empty
    row (energy from the embedding only, zero forces), against the reference step."""
    rng = np.random.default_rng(3)
    systems = [(np.zeros((1, 3)), [6]), (np.array([[0, 0, 0], [7.0, 0, 0]]), [1, 8]),
               (np.array([[0, 0, 0], [0, 6.0, 0], [0, 0, 12.0]]), [6, 7, 8]), (np.zeros((1, 3)), [1])]
    b = cases.pack(systems)
    B = len(systems)
    b["energy_mask"] = np.ones(B, np.uint8)
    b["force_mask"] = np.ones(B, np.uint8)
    b["energy"] = rng.normal(-3.0, 1.0, B)
    b["forces"] = rng.normal(0, 0.3, (int(b["atom_ptr"][-1]), 3))
    b["dataset_index"] = np.array([0, 1, 2, 0], np.int32)
    table = cases.random_table(cases.CFG[4], seed=4)
    params = oracle_ref.init_params(cases.CFG, 8)
    tc = pk.TrainConfig(seed=9, clip_norm=1e9)
    ref = oracle_ref.train_step(cases.CFG, 1, B, b, table, params, np.zeros_like(params), noise_sigma=tc.noise_sigma,
                                noise_scheme=1, seed=tc.seed, step=2, clip=tc.clip_norm)
    dev = pk.Device(_mcfg(pk), seed=0)
    dev.set_params(params)
    dev.set_rms_state(np.zeros_like(params))
    dev.set_reference_table(table)
    res = dev.train_step(b, tc, step=2)
    assert res.n_edges == 0
    assert abs(res.loss - ref["loss"]) <= TOL * abs(ref["loss"])
    assert abs(res.grad_norm - ref["grad_norm"]) <= TOL * ref["grad_norm"]
    assert_close(dev.grads(), ref["grads"], what="edge-less step gradient")
    dev.close()


def test_unlabeled_batch_is_a_zero_step(pk, oracle_ref):
    """No sample carries an energy or force label (both mask sums empty): the loss
    and gradient are zero, the RMS state decays, the parameters stay (S/loss.cpp:190-212,
    S/trainer.cpp:37-53) - as in the reference step."""
    b = cases.molecules(pk, 5, 21)
    B = len(b["atom_ptr"]) - 1
    b["energy_mask"] = np.zeros(B, np.uint8)
    b["force_mask"] = np.zeros(B, np.uint8)
    b["denoise"] = np.zeros(B, np.uint8)
    params = oracle_ref.init_params(cases.CFG, 5)
    v0 = np.full_like(params, 1e-4)
    tc = pk.TrainConfig(seed=2, clip_norm=10.0)
    table = cases.random_table(cases.CFG[4], seed=6)
    ref = oracle_ref.train_step(cases.CFG, 1, B, b, table, params, v0, noise_sigma=tc.noise_sigma, noise_scheme=1,
                                seed=tc.seed, step=0, clip=tc.clip_norm)
    dev = pk.Device(_mcfg(pk), seed=0)
    dev.set_params(params)
    dev.set_rms_state(v0)
    dev.set_reference_table(table)
    res = dev.train_step(b, tc, step=0)
    assert res.loss == 0.0 and ref["loss"] == 0.0
    assert res.grad_norm == 0.0 and ref["grad_norm"] == 0.0
    assert not np.any(dev.grads())
    assert np.array_equal(dev.params(), params)
    assert np.array_equal(dev.rms_state(), ref["rms_v"])
    dev.close()


def test_resume_from_checkpoint_is_bit_identical(pk, tmp_path):
    """Checkpoint / resume: parameters (LAMMCKPT, S/model.cpp:445-497) and the RMS
    state (LAMMRMS1) saved after step 1 and loaded into a new context reproduce the
    uninterrupted run's steps 2 and 3 bit for bit (pipelined staged steps)."""
    from paper_2505_22208_b200 import io
    mcfg = _mcfg(pk)
    batches = [cases.mixed_batch(pk, D=cases.CFG[4], seed=40 + s, count=12) for s in range(3)]
    table = cases.random_table(cases.CFG[4], seed=3)
    tc = pk.TrainConfig(seed=13)

    def run(dev, steps):
        for s in steps:
            dev.stage(batches[s], tc, step=s, slot=s)
        out = []
        for k, s in enumerate(steps):
            nxt = steps[k + 1] if k + 1 < len(steps) else None
            out.append(dev.train_step_staged(s, sync=True, next_slot=nxt))
        return out

    a = pk.Device(mcfg, seed=4)
    a.set_reference_table(table)
    run(a, [0])
    io.save_checkpoint(str(tmp_path / "p.ckpt"), mcfg, a.params())
    io.save_rms_state(str(tmp_path / "v.rms"), mcfg, a.rms_state())
    ra = run(a, [1, 2])
    pa, va = a.params(), a.rms_state()
    a.close()

    c1, p = io.load_checkpoint(str(tmp_path / "p.ckpt"))
    c2, v = io.load_rms_state(str(tmp_path / "v.rms"))
    assert c1 == mcfg and c2 == mcfg
    b = pk.Device(mcfg, seed=99)  # different init: everything comes from the files
    b.set_params(p)
    b.set_rms_state(v)
    b.set_reference_table(table)
    rb = run(b, [1, 2])
    assert [r.loss for r in ra] == [r.loss for r in rb]
    assert np.array_equal(pa.view(np.uint64), b.params().view(np.uint64))
    assert np.array_equal(va.view(np.uint64), b.rms_state().view(np.uint64))
    b.close()
