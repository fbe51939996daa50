"""GPU parity: liblamm_b200.so (sm_100a) through its C ABI vs the CPU oracle.

Bars: neighbour lists bit-exact (pair set, order, fp64 distance
and unit); energies, forces, loss and every gradient tensor within 1e-4 per
tensor (max|d|/max|ref| and ||d||/||ref||) in fp32 against the fp64 oracle;
the RMS optimizer bit-exact in fp64 given the same gradient.
"""
import numpy as np
import pytest

from conftest import TOL, assert_close, has_gpu, rel_err
import cases

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]




def tensors(cfg, flat):
    """Splits a flat parameter/gradient vector in for_each_tensor order."""
    H, L, K, _, D = cfg
    sizes = [("embedding", 118 * H)] + [(f"filter{l}", H * K) for l in range(L)] + \
            [(f"update{l}", H * H) for l in range(L)] + [("energy_head", H * D), ("force_head", (2 * H + K) * D)]
    out, o = {}, 0
    for name, n in sizes:
        out[name] = flat[o:o + n]
        o += n
    return out


def check_nlist(dev, oracle_ref, batch):
    dev.set_batch(batch)
    ptr, oi, oj, dist, unit = dev.build_neighbor_list()
    ap = batch["atom_ptr"]
    for s in range(len(ap) - 1):
        lo, hi = ap[s], ap[s + 1]
        ri, rj, rd, ru = oracle_ref.neighbor_list(batch["pos"][lo:hi], batch["Z"][lo:hi], 5.0)
        sl = slice(ptr[s], ptr[s + 1])
        assert np.array_equal(oi[sl], ri) and np.array_equal(oj[sl], rj), f"pair set/order differs in sample {s}"
        assert np.array_equal(dist[sl].view(np.uint64), rd.view(np.uint64)), f"fp64 distance bits differ ({s})"
        assert np.array_equal(unit[sl].view(np.uint64), ru.view(np.uint64)), f"fp64 unit bits differ ({s})"
    return ptr


def test_neighbor_list_bit_exact_molecules(pk, dev, oracle_ref):
    check_nlist(dev, oracle_ref, cases.molecules(pk, 64, 42))


def test_neighbor_list_edge_cases(pk, dev, oracle_ref):
    rng = np.random.default_rng(0)
    batch = cases.pack(cases.edge_systems(rng))
    ptr = check_nlist(dev, oracle_ref, batch)
    counts = np.diff(ptr)
    assert counts[0] == 0 and counts[1] == 2 and counts[2] == 0 and counts[3] == 0 and counts[4] == 2
    assert counts[5] == 0  # (0,0,0)-(3,4,0) and (0,0,0)-(0,0,5) are exactly 5 A: excluded


def test_neighbor_list_large_cluster(pk, dev, oracle_ref):
    # max-size samples: 2000-atom cluster next to small ones (ragged rows)
    big = pk.synth_generate(1, 3, mode=2000, sigma=0.01, min_atoms=2000, max_atoms=2000, elements=(14,),
                            relax_steps=0)
    small = cases.molecules(pk, 5, 9)
    check_nlist(dev, oracle_ref, pk.concat([small, big]))


def test_neighbor_list_cell_list_cases(pk, dev, oracle_ref):
    """Samples above kSmallAtoms (128) go through the cell lists: lattices whose
    pair distances sit exactly at the cutoff and at cell boundaries, degenerate
    extents (a line, one point), the 128/129 threshold, several 1024-atom windows,
    and a huge extent (the one-cell fallback)."""
    rng = np.random.default_rng(7)
    g = np.arange(6) * 2.5  # 6^3 lattice, spacing rc/2: pairs at exactly 5 A excluded
    lat = np.array([[a, b, c] for a in g for b in g for c in g], float)
    g5 = np.arange(5) * 5.0  # spacing rc: every nearest-neighbour distance is exactly the cutoff
    lat5 = np.array([[a, b, c] for a in g5 for b in g5 for c in g5], float) + 1e-3 * (rng.random((125, 3)) < 0.5)
    systems = [
        (lat, rng.choice(cases.ORGANIC, len(lat))),
        (lat5, rng.choice(cases.ORGANIC, 125)),
        (np.c_[np.arange(300) * 1.0, np.zeros(300), np.zeros(300)], np.full(300, 6)),  # a line
        (np.zeros((150, 3)), np.full(150, 1)),                                          # one point
        (rng.uniform(0, 12, (128, 3)), rng.choice(cases.ORGANIC, 128)),                 # threshold
        (rng.uniform(0, 12, (129, 3)), rng.choice(cases.ORGANIC, 129)),
        (rng.uniform(0, 32, (3000, 3)), rng.choice(cases.ORGANIC, 3000)),               # 3 windows
        (np.r_[rng.uniform(0, 1e8, (140, 3)), rng.uniform(0, 6, (20, 3))], np.full(160, 8)),  # huge extent
    ]
    mixed = pk.concat([cases.molecules(pk, 3, 4), cases.pack(systems), cases.molecules(pk, 2, 5)])
    ptr = check_nlist(dev, oracle_ref, mixed)
    assert np.diff(ptr)[3 + 3] == 150 * 149


def test_forward_matches_oracle(pk, dev, oracle_port):
    batch = cases.molecules(pk, 48, 11)
    params = oracle_port.init_params(cases.CFG, 7)
    dev.set_params(params)
    dev.set_batch(batch)
    e, f = dev.forward()
    re, rf = oracle_port.forward(cases.CFG, params, batch)
    assert_close(e, re, what="energy")
    assert_close(f, rf, what="forces")
    # ForwardCache of one sample (h per layer, tanh(m) per layer)
    ap = batch["atom_ptr"]
    h, mt = oracle_port.forward_cache(cases.CFG, params, batch["pos"][ap[0]:ap[1]], batch["Z"][ap[0]:ap[1]])
    for l in range(cases.CFG[1] + 1):
        assert_close(dev.forward_cache("h", l)[ap[0]:ap[1]], h[l], what=f"h[{l}]")
    for l in range(cases.CFG[1]):
        assert_close(dev.forward_cache("mu", l)[ap[0]:ap[1]], mt[l], what=f"tanh(m)[{l}]")


def test_forward_momentum_conservation(pk, dev):
    batch = cases.molecules(pk, 16, 12)
    dev.set_params(pk.init_params(dev.cfg, 3))
    dev.set_batch(batch)
    _, f = dev.forward()
    D, ap = dev.cfg.heads, batch["atom_ptr"]
    for s in range(len(ap) - 1):
        blk = f[3 * D * ap[s]:3 * D * ap[s + 1]].reshape(D, -1, 3)
        scale = np.abs(blk).max() + 1e-30
        assert np.abs(blk.sum(axis=1)).max() / scale < 1e-4


def test_loss_grad_matches_oracle(pk, dev, oracle_port):
    batch = cases.with_heads(cases.molecules(pk, 40, 13), cases.CFG[4], seed=1)
    batch["energy_mask"][::3] = 0
    batch["force_mask"][::4] = 0
    params = oracle_port.init_params(cases.CFG, 5)
    dev.set_params(params)
    dev.set_reference_table(None)
    dev.set_batch(batch)
    bd, ge, gf = dev.masked_loss_grad()
    pe, pf = oracle_port.forward(cases.CFG, params, batch)
    rbd, rge, rgf = oracle_port.loss_grad(batch, cases.CFG[4], pe, pf)
    for k in ("total", "energy_term", "force_term"):
        assert abs(bd[k] - rbd[k]) <= TOL * max(abs(rbd[k]), 1e-12), k
    assert bd["energy_labeled"] == rbd["energy_labeled"] and bd["force_labeled"] == rbd["force_labeled"]
    assert np.array_equal(np.sign(ge), np.sign(rge))
    assert_close(ge, rge, what="dL/dE")
    assert_close(gf, rgf, what="dL/dF")


def test_backward_general_upstream(pk, dev, oracle_port):
    batch = cases.molecules(pk, 24, 14)
    params = oracle_port.init_params(cases.CFG, 9)
    rng = np.random.default_rng(3)
    ap = batch["atom_ptr"]
    up_e = rng.normal(size=(len(ap) - 1, cases.CFG[4]))
    up_f = rng.normal(size=3 * cases.CFG[4] * int(ap[-1]))
    dev.set_params(params)
    dev.set_batch(batch)
    g = dev.backward(up_e, up_f)
    rg = oracle_port.backward(cases.CFG, params, batch, up_e, up_f)
    for name, t in tensors(cases.CFG, g).items():
        assert_close(t, tensors(cases.CFG, rg)[name], what=f"d/d{name}")


def test_backward_accumulates(pk, dev, oracle_port):
    batch = cases.molecules(pk, 8, 15)
    dev.set_batch(batch)
    rng = np.random.default_rng(4)
    ue = rng.normal(size=(8, cases.CFG[4]))
    uf = rng.normal(size=3 * cases.CFG[4] * int(batch["atom_ptr"][-1]))
    g1 = dev.backward(ue, uf)
    g2 = dev.backward(ue, uf, grads=g1.copy())
    assert np.allclose(g2, 2 * g1, rtol=1e-6, atol=1e-12)
    zero = dev.backward(np.zeros_like(ue), np.zeros_like(uf))
    assert not np.any(zero)  # SPEC: zero loss gradient in -> zero parameter gradient out


def _train_cfg(pk, **kw):
    return pk.TrainConfig(seed=kw.pop("seed", 17), **kw)


def test_train_step_matches_oracle(pk, oracle_ref):
    """One full step (denoise -> normalize -> fwd -> per-rank loss -> bwd -> /G -> clip -> RMS)."""
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    dev = pk.Device(mcfg, seed=0)
    params = oracle_ref.init_params(cases.CFG, 21)
    batch = cases.mixed_batch(pk, D=cases.CFG[4], seed=5, count=24)
    table = cases.random_table(cases.CFG[4], seed=2)
    tc = _train_cfg(pk, clip_norm=1e9)
    v0 = np.zeros_like(params)
    ref = oracle_ref.train_step(cases.CFG, 1, 24, batch, table, params, v0, noise_sigma=tc.noise_sigma,
                                noise_scheme=1, seed=tc.seed, step=3, clip=tc.clip_norm)
    dev.set_params(params)
    dev.set_rms_state(v0)
    dev.set_reference_table(table)
    res = dev.train_step(batch, tc, step=3, workers=1, rank=0)
    assert abs(res.loss - ref["loss"]) <= TOL * abs(ref["loss"])
    assert abs(res.grad_norm - ref["grad_norm"]) <= TOL * ref["grad_norm"]
    g = dev.grads()
    for name, t in tensors(cases.CFG, g).items():
        assert_close(t, tensors(cases.CFG, ref["grads"])[name], what=f"step d/d{name}")
    # RMS state after one step from v=0 is 0.01 g^2: relative parity of g^2
    assert_close(dev.rms_state(), ref["rms_v"], tol=3 * TOL, what="rms v")
    dev.close()


@pytest.mark.parametrize("cfg", [(64, 2, 16, 5.0, 3), (32, 1, 8, 4.0, 3), (64, 2, 8, 4.5, 2), (32, 2, 16, 5.0, 1),
                                 (128, 2, 8, 5.0, 3)])
def test_train_step_other_model_sizes(pk, oracle_ref, cfg):
    """The other device instantiations through a full step, with samples above the
    cell-list threshold: hidden 64 / 32 (unfused update backward + split-K dW_u GEMM,
    FFMA filter) and hidden 128 with 8 Gaussians (the tensor-core filter with one
    K-step, the fused layer and update-backward kernels); the reference's
    own default is hidden 64 / rbf 16 / 2 layers / 1 head."""
    mcfg = pk.ModelConfig(*cfg[:3], cutoff=cfg[3], heads=cfg[4])
    dev = pk.Device(mcfg, seed=0)
    params = oracle_ref.init_params(cfg, 21)
    big = pk.synth_generate(2, 3, mode=300, sigma=0.01, min_atoms=290, max_atoms=310, elements=(6, 8))
    batch = cases.with_heads(pk.concat([cases.mixed_batch(pk, D=cfg[4], seed=9, count=12), big]), cfg[4], seed=4)
    batch["energy_mask"][:] = 1
    B = len(batch["atom_ptr"]) - 1
    table = cases.random_table(cfg[4], seed=2)
    tc = _train_cfg(pk, clip_norm=1e9)
    v0 = np.zeros_like(params)
    ref = oracle_ref.train_step(cfg, 1, B, batch, table, params, v0, noise_sigma=tc.noise_sigma,
                                noise_scheme=1, seed=tc.seed, step=1, clip=tc.clip_norm)
    dev.set_params(params)
    dev.set_rms_state(v0)
    dev.set_reference_table(table)
    res = dev.train_step(batch, tc, step=1, workers=1, rank=0)
    assert abs(res.loss - ref["loss"]) <= TOL * abs(ref["loss"])
    for name, t in tensors(cfg, dev.grads()).items():
        assert_close(t, tensors(cfg, ref["grads"])[name], what=f"{cfg[0]}: step d/d{name}")
    dev.close()


def test_denoise_labels_match_reference(pk, oracle_ref):
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    dev = pk.Device(mcfg, seed=0)
    batch = cases.mixed_batch(pk, D=cases.CFG[4], seed=8, count=12)
    table = cases.random_table(cases.CFG[4], seed=3)
    dev.set_reference_table(table)
    tc = _train_cfg(pk)
    B, G, rank, step = 12, 3, 2, 5
    dev.set_option("rank_local", 1)  # one rank's share without a communicator
    dev.train_step(batch, tc, step=step, workers=G, rank=rank)
    # worker-major position of sample b on rank r is r*B + b (S/trainer.cpp:268)
    e_dev, f_dev = dev.labels()
    ap = batch["atom_ptr"]
    for s in np.nonzero(batch["denoise"])[0]:
        seed = oracle_ref.mix_seed(oracle_ref.mix_seed(tc.seed, 0x4e4f4953 + step), rank * B + s)
        noisy, lab = oracle_ref.apply_noise(batch["pos"][ap[s]:ap[s + 1]], batch["Z"][ap[s]:ap[s + 1]], 0.3, 1, seed)
        d = batch["dataset_index"][s]
        assert np.array_equal(f_dev[ap[s]:ap[s + 1]], (1.0 / table["fstd"][d]) * lab), f"denoise labels {s}"
    dev.close()


def test_optimizer_bit_exact(pk, dev, oracle_ref):
    rng = np.random.default_rng(6)
    params = oracle_ref.init_params(cases.CFG, 4)
    v = rng.uniform(0, 1e-3, len(params))
    g = rng.normal(size=len(params)) * 1e-2
    tc = pk.TrainConfig(clip_norm=1e9)
    dev.set_params(params)
    dev.set_rms_state(v)
    dev.optimizer_step(g * 2, 2, tc)  # worker-summed grads, G = 2
    gs = g * 2 * (1.0 / 2)
    vv = 0.99 * v + (1.0 - 0.99) * gs * gs
    pp = params - 1e-3 * gs / (np.sqrt(vv) + 1e-8)
    assert np.array_equal(dev.rms_state().view(np.uint64), vv.view(np.uint64))
    assert np.array_equal(dev.params().view(np.uint64), pp.view(np.uint64))


def test_train_step_deterministic(pk):
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    batch = cases.mixed_batch(pk, D=cases.CFG[4], seed=9, count=32)
    table = cases.random_table(cases.CFG[4], seed=1)
    outs = []
    for _ in range(2):
        dev = pk.Device(mcfg, seed=3)
        dev.set_reference_table(table)
        for step in range(3):
            dev.train_step(batch, _train_cfg(pk), step=step)
        outs.append(dev.params())
        dev.close()
    assert np.array_equal(outs[0], outs[1])


def test_multi_worker_sum_semantics(pk, oracle_ref):
    """G simulated workers: per-rank loss/grad on one GPU == the reference's G-worker step."""
    G, B = 2, 8
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    params = oracle_ref.init_params(cases.CFG, 2)
    batch = cases.mixed_batch(pk, D=cases.CFG[4], seed=12, count=G * B)
    table = cases.random_table(cases.CFG[4], seed=4)
    tc = _train_cfg(pk, clip_norm=1e9)
    ref = oracle_ref.train_step(cases.CFG, G, B, batch, table, params, np.zeros_like(params), seed=tc.seed,
                                step=1, clip=tc.clip_norm)
    gsum = np.zeros_like(params)
    loss = 0.0
    for r in range(G):
        dev = pk.Device(mcfg, seed=0)
        dev.set_params(params)
        dev.set_reference_table(table)
        dev.set_option("rank_local", 1)
        shard = pk.select(batch, np.arange(r * B, (r + 1) * B))
        res = dev.train_step(shard, tc, step=1, workers=G, rank=r)
        gsum += dev.grads()
        loss += res.local["total"]
        dev.close()
    assert abs(loss / G - ref["loss"]) <= TOL * abs(ref["loss"])
    assert_close(gsum / G, ref["grads"], what="G-worker mean gradient")
    assert rel_err(gsum / G, ref["grads"])[0] < TOL


def test_simulated_workers_step_matches_reference(pk, oracle_ref):
    """lamm_train_step_workers: G simulated workers in worker order on one device,
    fp64 gradient sum, one optimizer step == the reference's step (S/trainer.cpp:262-326),
    denoising draws at positions g*B + b included."""
    G, B = 3, 6
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    params = oracle_ref.init_params(cases.CFG, 8)
    batch = cases.mixed_batch(pk, D=cases.CFG[4], seed=31, count=G * B)
    table = cases.random_table(cases.CFG[4], seed=6)
    tc = _train_cfg(pk, clip_norm=1e9)
    v0 = np.zeros_like(params)
    ref = oracle_ref.train_step(cases.CFG, G, B, batch, table, params, v0, seed=tc.seed, step=4,
                                clip=tc.clip_norm)
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_rms_state(v0)
    dev.set_reference_table(table)
    shards = [pk.select(batch, np.arange(g * B, (g + 1) * B)) for g in range(G)]
    res = dev.train_step_workers(shards, tc, step=4)
    assert res.n_atoms == int(batch["atom_ptr"][-1])
    assert abs(res.loss - ref["loss"]) <= TOL * abs(ref["loss"])
    assert abs(res.grad_norm - ref["grad_norm"]) <= TOL * ref["grad_norm"]
    assert_close(dev.rms_state(), ref["rms_v"], tol=3 * TOL, what="rms v after the G-worker step")
    assert_close(dev.grads() / G, ref["grads"], what="worker-summed gradient / G")
    # a second step continues from the device state (graph reuse, accumulator reset)
    ref2 = oracle_ref.train_step(cases.CFG, G, B, batch, table, ref["params"], ref["rms_v"], seed=tc.seed, step=5,
                                 clip=tc.clip_norm)
    dev.set_params(ref["params"])
    dev.set_rms_state(ref["rms_v"])
    res2 = dev.train_step_workers(shards, tc, step=5)
    assert abs(res2.loss - ref2["loss"]) <= TOL * abs(ref2["loss"])
    assert abs(res2.grad_norm - ref2["grad_norm"]) <= TOL * ref2["grad_norm"]
    dev.close()


def test_nccl_allreduce_path_single_rank(pk):
    """The data-parallel path on one rank: a real one-rank NCCL communicator, the
    ncclAllReduce captured inside the single step graph (and issued between the two
    graphs of the profiling pass): identical to the communicator-free step, bit for bit."""
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    batch = cases.mixed_batch(pk, D=cases.CFG[4], seed=17, count=16)
    table = cases.random_table(cases.CFG[4], seed=6)
    outs = []
    for use_comm in (False, True):
        dev = pk.Device(mcfg, seed=5)
        dev.set_reference_table(table)
        if use_comm:
            dev.comm_init(1, 0, pk.comm_unique_id())
        res = [dev.train_step(batch, _train_cfg(pk), step=s) for s in range(2)]
        dev.stage(batch, _train_cfg(pk), step=2, slot=0)
        res.append(dev.train_step_staged(0, sync=True))
        res += dev.train_steps_pipelined([batch, batch], _train_cfg(pk), [3, 4])  # submit/wait with NCCL
        dev.set_option("profile", 1)  # the per-kernel-event pass: two graphs, the allreduce between them
        res.append(dev.train_step(batch, _train_cfg(pk), step=5))
        dev.set_option("profile", 0)
        if use_comm:  # the captured allreduce ran: this rank's pre-allreduce time is recorded
            res.append(dev.train_step(batch, _train_cfg(pk), step=6))
            assert 0.0 < dev.last_step_compute_ms() < 1e3
        else:
            res.append(dev.train_step(batch, _train_cfg(pk), step=6))
            with pytest.raises(pk.InputError):
                dev.last_step_compute_ms()
        outs.append((dev.params(), dev.grads(), [r.loss for r in res]))
        dev.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


def test_evaluate_matches_reference(pk, oracle_ref):
    """trainer::evaluate (S/trainer.cpp:528-553): physical-unit MAEs of the
    current parameters, each sample's own head denormalized with the table."""
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    params = oracle_ref.init_params(cases.CFG, 13)
    batch = cases.mixed_batch(pk, D=cases.CFG[4], seed=21, count=40)
    batch["denoise"][:] = 0
    table = cases.random_table(cases.CFG[4], seed=9)
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_reference_table(table)
    got = dev.evaluate(batch)
    want = oracle_ref.evaluate(cases.CFG, params, batch, table)
    dev.close()
    assert got["energy_count"] == want["energy_count"] and got["force_count"] == want["force_count"]
    for k in ("energy_mae", "force_mae"):
        assert abs(got[k] - want[k]) <= TOL * abs(want[k]), (k, got[k], want[k])


@pytest.mark.parametrize("denoise", [False, True])
def test_train_step_large_structures(pk, oracle_ref, denoise):
    """cfg4-like: two 500-700 atom clusters (dense lists, ~30+ edges per atom,
    partitions cutting through one atom's row run) through the full step; with
    denoise, the second cluster is a coordinate-denoising sample (its centered
    noise mean staged through shared memory, cell lists over the noisy positions)."""
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    batch = cases.synth(pk, 2, 77, mode=600, sigma=0.1, min_atoms=500, max_atoms=700, elements=cases.ORGANIC)
    batch = cases.with_heads(batch, cases.CFG[4], seed=3)
    if denoise:
        batch["denoise"][1] = 1
    table = cases.random_table(cases.CFG[4], seed=12)
    params = oracle_ref.init_params(cases.CFG, 31)
    tc = _train_cfg(pk, clip_norm=1e9)
    ref = oracle_ref.train_step(cases.CFG, 1, 2, batch, table, params, np.zeros_like(params), seed=tc.seed, step=0,
                                clip=tc.clip_norm)
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_rms_state(np.zeros_like(params))
    dev.set_reference_table(table)
    res = dev.train_step(batch, tc, step=0)
    assert res.n_edges > 25 * res.n_atoms
    assert abs(res.loss - ref["loss"]) <= TOL * abs(ref["loss"])
    g = dev.grads()
    for name, t in tensors(cases.CFG, g).items():
        assert_close(t, tensors(cases.CFG, ref["grads"])[name], what=f"large d/d{name}")
    dev.close()


def test_staged_steps_match_host_steps(pk):
    """Device-resident staged slots of different sizes replayed through one
    captured graph give the same trajectory as host-batch steps."""
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    batches = [cases.mixed_batch(pk, D=cases.CFG[4], seed=40 + k, count=n) for k, n in enumerate((24, 8, 40))]
    table = cases.random_table(cases.CFG[4], seed=5)
    tc = _train_cfg(pk)
    outs = []
    for staged in (False, True):
        dev = pk.Device(mcfg, seed=8)
        dev.set_reference_table(table)
        if staged:
            for k, b in enumerate(batches):
                dev.stage(b, tc, step=k, slot=k)
        losses = []
        for rep in range(2):
            for k, b in enumerate(batches):
                step = k  # the staged slot carries its step's denoise draws
                r = dev.train_step_staged(k, sync=True) if staged else dev.train_step(b, tc, step=step)
                losses.append(r.loss)
        outs.append((dev.params(), losses))
        dev.close()
    assert outs[0][1] == outs[1][1]
    assert np.array_equal(outs[0][0], outs[1][0])


def _pipeline_vs_sync(pk, batches, table=None):
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    tc = _train_cfg(pk)
    outs = []
    for piped in (False, True):
        dev = pk.Device(mcfg, seed=8)
        if table is not None:
            dev.set_reference_table(table)
        steps = list(range(len(batches)))
        if piped:
            rs = dev.train_steps_pipelined(batches, tc, steps)
        else:
            rs = [dev.train_step(b, tc, step=k) for k, b in zip(steps, batches)]
        outs.append((dev.params(), [(r.loss, r.grad_norm, r.n_atoms, r.n_edges) for r in rs], dev.anomalies()))
        dev.close()
    return outs


def test_pipelined_steps_match_sync(pk):
    """lamm_train_step_submit/_wait (host packs step k+1 while the device runs
    step k) reproduces the synchronous trajectory bit for bit."""
    batches = [cases.mixed_batch(pk, D=cases.CFG[4], seed=60 + k, count=n) for k, n in enumerate((24, 8, 40, 16, 30))]
    outs = _pipeline_vs_sync(pk, batches, cases.random_table(cases.CFG[4], seed=5))
    assert outs[0][1] == outs[1][1]
    assert np.array_equal(outs[0][0], outs[1][0])


def test_pipelined_overflow_reruns_the_chain(pk):
    """A step that overflows the edge capacity while the next one is already in
    flight: the device skips the next step's update, the wait reruns both in
    order, and the trajectory equals the synchronous one."""
    rng = np.random.default_rng(3)
    mol = [cases.molecules(pk, 6, 70 + k) for k in range(3)]
    dense = [cases.pack([(rng.uniform(0, 4, (150, 3)), np.full(150, 6))]) for _ in range(2)]
    for b in dense:
        b["energy_mask"][:] = 1
        b["energy"][:] = -100.0
    batches = [mol[0], dense[0], mol[1], dense[1], mol[2]]
    outs = _pipeline_vs_sync(pk, batches)
    assert outs[0][1] == outs[1][1]
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[1][1][1][3] > 32 * 150  # the dense step did exceed the first capacity guess


def test_sync_step_refused_while_pipelined(pk):
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    dev = pk.Device(mcfg, seed=8)
    tc = _train_cfg(pk)
    b = cases.molecules(pk, 4, 1)
    t = dev.train_step_submit(b, tc, 0)
    with pytest.raises(pk.InputError):
        dev.train_step(b, tc, step=1)
    with pytest.raises(pk.InputError):
        dev.params()  # device state is not read mid-flight
    with pytest.raises(pk.InputError):
        dev.train_step_wait(t + 1)
    assert np.isfinite(dev.train_step_wait(t).loss)
    dev.close()


def test_staged_next_prefetch_is_bit_identical(pk):
    """lamm_train_step_staged_next: each step's batch preparation (prep + neighbour
    list) built ahead on a side stream into the other batch-state parity while the
    previous step's model runs. Slots of different kinds (molecules, a cell-list
    batch, periodic image cells, a dense batch that overflows the first edge
    capacity guess mid-pipeline) cycled twice: parameters, RMS state and every loss
    equal the unpipelined staged steps bit for bit."""
    import test_periodic
    rng = np.random.default_rng(9)
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    big = cases.molecules(pk, 3, 4)
    pos, Z, cell = cases.diamond_supercell(reps=3, seed=2)  # 216 atoms: cell lists
    n = len(Z)
    big = pk.concat([big, dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z, forces=rng.normal(0, 0.1, (n, 3)),
                                dataset_index=np.zeros(1, np.int32), energy_mask=np.ones(1, np.uint8),
                                force_mask=np.ones(1, np.uint8), energy=np.array([-4.6 * n]),
                                denoise=np.zeros(1, np.uint8))])
    dense = cases.pack([(rng.uniform(0, 4, (150, 3)), np.full(150, 6))])
    dense["energy_mask"][:] = 1
    dense["energy"][:] = -100.0
    slots = [cases.mixed_batch(pk, D=cases.CFG[4], seed=40, count=12), big, test_periodic.image_batch(pk, seed=3),
             dense, cases.mixed_batch(pk, D=cases.CFG[4], seed=41, count=20)]
    table = cases.random_table(cases.CFG[4], seed=2, elements=(1, 6, 7, 8, 14))
    outs = []
    for pipelined in (False, True):
        dev = pk.Device(mcfg, seed=5)
        dev.set_reference_table(table)
        tc = _train_cfg(pk)
        for k, b in enumerate(slots):
            dev.stage(b, tc, step=k, slot=k)
        order = [0, 1, 2, 3, 4, 2, 0, 4, 1, 3]
        losses = []
        for t, k in enumerate(order):
            nxt = order[t + 1] if pipelined and t + 1 < len(order) else None
            r = dev.train_step_staged(k, sync=True, next_slot=nxt)
            losses.append((r.loss, r.grad_norm, r.n_edges))
        outs.append((dev.params(), dev.rms_state(), losses))
        dev.close()
    assert outs[0][2] == outs[1][2]
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
