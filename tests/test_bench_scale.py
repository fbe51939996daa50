"""GPU parity at the sizes BASELINE.json names, through the paths bench.py times.

* cfg2 (configs[1]): the exact staged slots bench.py builds (256 molecules,
  ~7.4k atoms, ~131k directed edges per step, balanced plan), run with
  train_step_staged — the headline's own call — against the reference step
  (oracle/_ref, S/trainer.cpp:258-327). The edge kernels' steady-state TMA
  restaging (a group walking >= 3 staged chunks, edge_kernels.cuh walk_edges)
  is asserted to be exercised, computed from the CSR exactly as the device cuts it.
* cfg3 (configs[2]): the semi-supervised mix (E+F / energy-only / denoising
  subsets, 8-200 atoms, T = 2 epoch index), one balanced mini-batch at G = 8,
  B = 32 through lamm_train_step_workers vs the reference's G-worker step.
* cfg4 (configs[3]): B = 4 diamond-Si supercells of 216-1000 atoms (28 neighbours
  per atom): the non-periodic twin vs oracle/_ref, the periodic batch vs the port.

Bars: per tensor max-rel and L2-rel <= 1e-4 (fp32 vs fp64).
"""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, TOL, assert_close, has_gpu
import cases

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

THREADS = os.cpu_count() or 8


def _tensors(cfg, flat):
    H, L, K, _, D = cfg
    sizes = [("embedding", 118 * H)] + [(f"filter{l}", H * K) for l in range(L)] + \
            [(f"update{l}", H * H) for l in range(L)] + [("energy_head", H * D), ("force_head", (2 * H + K) * D)]
    out, o = {}, 0
    for name, n in sizes:
        out[name] = flat[o:o + n]
        o += n
    return out


def _check_step(res, grads, rms_v, ref, cfg, what):
    assert abs(res.loss - ref["loss"]) <= TOL * abs(ref["loss"]), (what, res.loss, ref["loss"])
    assert abs(res.grad_norm - ref["grad_norm"]) <= TOL * ref["grad_norm"], (what, res.grad_norm, ref["grad_norm"])
    rg = _tensors(cfg, ref["grads"])
    for name, t in _tensors(cfg, grads).items():
        assert_close(t, rg[name], what=f"{what}: d/d{name}")
    if rms_v is not None:
        assert_close(rms_v, ref["rms_v"], tol=3 * TOL, what=f"{what}: rms v")


def row_ptr_of(dev, batch):
    """Global CSR row offsets of the batch's neighbour list (device-built, bit-exact)."""
    dev.set_batch(batch)
    ptr, oi, _, _, _ = dev.build_neighbor_list(fp64=False)
    ap = batch["atom_ptr"]
    N = int(ap[-1])
    counts = np.zeros(N, np.int64)
    for s in range(len(ap) - 1):
        np.add.at(counts, oi[ptr[s]:ptr[s + 1]] + ap[s], 1)
    return np.concatenate([[0], np.cumsum(counts)])


def max_chunks_per_group(row_ptr, Q, groups, parts_per_cta, block, chunk, atom_cost):
    """Replays k_nbr_fill's cost-balanced cut (x_i = row_ptr[i] + atom_cost i,
    T = P + atom_cost N, part_lo[q] = first atom with x_i >= floor(T q / Q),
    kernels.cuh) and walk_edges' chunking (chunks start on whole blocks): the largest
    number of staged chunks any group walks."""
    N, P = len(row_ptr) - 1, int(row_ptr[-1])
    T = P + atom_cost * N
    part_lo = np.zeros(Q + 1, np.int64)
    part_lo[Q] = N
    for i in range(N):
        x = int(row_ptr[i]) + atom_cost * i
        qlo = 0 if i == 0 else ((int(row_ptr[i - 1]) + atom_cost * (i - 1) + 1) * Q + T - 1) // T
        qhi = min(((x + 1) * Q + T - 1) // T - 1, Q - 1)
        if qhi >= qlo:
            part_lo[qlo:qhi + 1] = i
        if i == N - 1:
            part_lo[((x + 1) * Q + T - 1) // T:Q] = N
    per = parts_per_cta // groups
    best = 0
    for q0 in range(0, Q, per):
        e0, e1 = int(row_ptr[part_lo[q0]]), int(row_ptr[part_lo[q0 + per]])
        if e1 > e0:
            base = e0 & ~(block - 1)
            best = max(best, (e1 - base + chunk - 1) // chunk)
    return best


def test_cfg2_bench_slots_match_reference(pk, oracle_ref):
    """The bench's own staged cfg2 slots (bench.make_workload), the heaviest and the
    lightest of the epoch, each run through train_step_staged from the same
    parameters/RMS state as the reference step."""
    sys.path.insert(0, ROOT)
    import bench
    pool, table, sched = bench.make_workload(pk, 1)
    mcfg = pk.ModelConfig(**bench.CFG)
    cfg = mcfg.astuple()
    from paper_2505_22208_b200.dist import shard
    shards = [shard(pool, sched, s, 0, 1, bench.BATCH_PER_GPU) for s in range(sched["n_batches"])]
    atoms = [int(b["atom_ptr"][-1]) for b in shards]
    picks = [int(np.argmax(atoms)), int(np.argmin(atoms))]
    params = oracle_ref.init_params(cfg, 7)
    v0 = np.random.default_rng(1).uniform(0.0, 1e-4, len(params))  # a warm RMS state
    tc = pk.TrainConfig(seed=11, clip_norm=1e9)
    dev = pk.Device(mcfg, seed=7)
    geo = {k: dev.info(k) for k in ("grid_edge", "parts_per_cta", "chunk_edges", "message_groups", "message_block",
                                    "edge_groups", "edge_block", "atom_cost")}
    Q = geo["grid_edge"] * geo["parts_per_cta"]
    for s in picks:
        b = shards[s]
        rp = row_ptr_of(dev, b)
        assert len(b["atom_ptr"]) - 1 == 256
        if s == picks[0]:  # the steady-state restage path (k + 2 < nchunks) runs
            assert atoms[s] > 5000
            for g, blk in ((geo["message_groups"], geo["message_block"]), (geo["edge_groups"], geo["edge_block"])):
                nch = max_chunks_per_group(rp, Q, g, geo["parts_per_cta"], blk, geo["chunk_edges"], geo["atom_cost"])
                assert nch >= 3, (g, blk, nch)
        ref = oracle_ref.train_step(cfg, 1, 256, b, table, params, v0, seed=tc.seed, step=s, clip=tc.clip_norm,
                                    threads=THREADS)
        dev.set_params(params)
        dev.set_rms_state(v0)
        dev.set_reference_table(table)
        dev.stage(b, tc, step=s, slot=s)
        res = dev.train_step_staged(s, sync=True)
        assert res.n_edges == int(rp[-1])
        _check_step(res, dev.grads(), dev.rms_state(), ref, cfg, f"cfg2 slot {s} ({atoms[s]} atoms, {res.n_edges} edges)")
    dev.close()


def test_cfg2_consecutive_staged_steps_match_reference(pk, oracle_ref):
    """Three consecutive headline steps exactly as bench.py runs them (graph replay,
    the next step's batch preparation built on the side stream during each step,
    parameters and RMS state carried on the device, the default clip of 10) against
    three reference steps."""
    sys.path.insert(0, ROOT)
    import bench
    pool, table, sched = bench.make_workload(pk, 1)
    mcfg = pk.ModelConfig(**bench.CFG)
    cfg = mcfg.astuple()
    from paper_2505_22208_b200.dist import shard
    tc = pk.TrainConfig(seed=11)
    params = oracle_ref.init_params(cfg, 7)
    v = np.zeros_like(params)
    dev = pk.Device(mcfg, seed=7)
    dev.set_params(params)
    dev.set_rms_state(v)
    dev.set_reference_table(table)
    for s in range(3):
        b = shard(pool, sched, s, 0, 1, bench.BATCH_PER_GPU)
        dev.stage(b, tc, step=s, slot=s)
    for s in range(3):
        b = shard(pool, sched, s, 0, 1, bench.BATCH_PER_GPU)
        ref = oracle_ref.train_step(cfg, 1, 256, b, table, params, v, seed=tc.seed, step=s, clip=tc.clip_norm,
                                    threads=THREADS)
        res = dev.train_step_staged(s, sync=True, next_slot=(s + 1) % 3)
        _check_step(res, dev.grads(), None, ref, cfg, f"cfg2 consecutive step {s}")
        params, v = ref["params"], ref["rms_v"]
        # continue both from the reference's state so fp32 drift does not compound
        dev.set_params(params)
        dev.set_rms_state(v)
    dev.close()


def test_cfg3_semisupervised_mix_g8_b32(pk, oracle_ref):
    """One balanced mini-batch of the LaMM semi-supervised mix at G = 8, B = 32 (256
    samples, three heads, ~1/3 denoising): the 8 workers simulated in worker order on
    the device (lamm_train_step_workers) vs the reference's 8-worker step."""
    subs = []
    for k, (task, mode, n) in enumerate((("energy_and_forces", 15.0, 400), ("energy_only", 60.0, 80),
                                         ("denoising", 30.0, 200))):
        subs.append(pk.synth_generate(n, 21 + k, task=task, mode=mode, sigma=0.5, min_atoms=8, max_atoms=200,
                                      elements=cases.ORGANIC, threads=THREADS, dataset_index=k))
    sizes = [len(b["atom_ptr"]) - 1 for b in subs]
    osub, osam = pk.build_epoch_index(pk.temperature_counts(sizes, 2.0), sizes, seed=5)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    pool = pk.select(pk.concat(subs), offs[osub] + osam)
    G, B = 8, 32
    sched = pk.plan(np.diff(pool["atom_ptr"]), G, B, 4, seed=3, mode="balanced")
    ids = sched["sample"][:G * B]
    batch = pk.select(pool, ids)
    assert batch["denoise"].sum() > 20 and len(set(batch["dataset_index"].tolist())) == 3
    D = cases.CFG[4]
    table = cases.random_table(D, seed=8)
    params = oracle_ref.init_params(cases.CFG, 3)
    v0 = np.zeros_like(params)
    tc = pk.TrainConfig(seed=19, clip_norm=1e9)
    ref = oracle_ref.train_step(cases.CFG, G, B, batch, table, params, v0, seed=tc.seed, step=2, clip=tc.clip_norm,
                                threads=THREADS)
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=D)
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_rms_state(v0)
    dev.set_reference_table(table)
    res = dev.train_step_workers([pk.select(batch, np.arange(g * B, (g + 1) * B)) for g in range(G)], tc, step=2)
    assert res.n_atoms == int(batch["atom_ptr"][-1])
    # grads_get after simulated workers: the fp64 worker sum the optimizer consumed (before /G)
    _check_step(res, dev.grads() / G, dev.rms_state(), ref, cases.CFG, "cfg3 G=8 B=32")
    dev.close()


def _supercell_batch(seed=11, B=4, periodic=True):
    """bench.supercells_cfg4's first B samples: r0 x r1 x r2 diamond-Si supercells,
    r in 3..5 (216-1000 atoms), labels from random values."""
    rng = np.random.default_rng(seed)
    parts = []
    for s in range(B):
        pos, Z, cell = cases.diamond_supercell(reps=tuple(rng.integers(3, 6, 3)), seed=1000 + s)
        n = len(Z)
        parts.append(dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z, forces=rng.normal(0, 0.1, (n, 3)),
                          dataset_index=np.zeros(1, np.int32), energy_mask=np.ones(1, np.uint8),
                          force_mask=np.ones(1, np.uint8), energy=np.array([-4.6 * n + rng.normal()]),
                          denoise=np.zeros(1, np.uint8), cell=cell[None] if periodic else None))
    return cases.lib_concat(parts)


def test_cfg4_supercells_nonperiodic_twin_vs_reference(pk, oracle_ref):
    batch = _supercell_batch(periodic=False)
    batch["dataset_index"] = np.array([0, 3, 5, 9], np.int32)
    assert 200 <= np.diff(batch["atom_ptr"]).min() and np.diff(batch["atom_ptr"]).max() <= 1000
    table = cases.random_table(cases.CFG[4], seed=4, elements=(14,))
    params = oracle_ref.init_params(cases.CFG, 17)
    tc = pk.TrainConfig(seed=5, clip_norm=1e9)
    ref = oracle_ref.train_step(cases.CFG, 1, 4, batch, table, params, np.zeros_like(params), seed=tc.seed, step=0,
                                clip=tc.clip_norm, threads=THREADS)
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_rms_state(np.zeros_like(params))
    dev.set_reference_table(table)
    res = dev.train_step(batch, tc, step=0)
    assert res.n_edges > 20 * res.n_atoms
    _check_step(res, dev.grads(), dev.rms_state(), ref, cases.CFG, "cfg4 non-periodic twin")
    dev.close()


def test_cfg4_periodic_supercells_vs_port(pk, oracle_port):
    """Periodic cfg4 batch (minimum image; parity-unpinned extension: the C port's
    minimum image is itself checked against a 27-image enumeration in test_periodic)."""
    batch = _supercell_batch(periodic=True)
    table = cases.random_table(cases.CFG[4], seed=4, elements=(14,))
    params = oracle_port.init_params(cases.CFG, 17)
    tc = pk.TrainConfig(seed=5, clip_norm=1e9)
    with oracle_port.periodic(batch["cell"]):
        ref = oracle_port.train_step(cases.CFG, 1, 4, batch, table, params, np.zeros_like(params), seed=tc.seed,
                                     step=0, clip=tc.clip_norm)
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4])
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_rms_state(np.zeros_like(params))
    dev.set_reference_table(table)
    res = dev.train_step(batch, tc, step=0)
    assert res.n_edges == 28 * res.n_atoms  # every Si has its 4 + 12 + 12 neighbours within 5 A
    _check_step(res, dev.grads(), dev.rms_state(), ref, cases.CFG, "cfg4 periodic")
    dev.close()


def test_cfg3_periodic_crystals_g8_b32_vs_port(pk, oracle_port):
    """The literal cfg3 (BASELINE configs[2]): periodic crystals of 8-200 atoms (4.6-14 A
    cells: the small ones need several images per pair), E+F / energy-only / denoising
    subsets mixed at T = 2, one balanced mini-batch at G = 8, B = 32 through the
    simulated-worker step vs the C port's G-worker step under the same cells
    (parity-unpinned extension; the port's images are checked in test_periodic)."""
    sys.path.insert(0, ROOT)
    import bench
    subs = [bench.crystal_pool(pk, n, 21 + k, task, mode, dataset_index=k)
            for k, (task, mode, n) in enumerate((("energy_and_forces", 15.0, 400), ("energy_only", 60.0, 80),
                                                 ("denoising", 30.0, 200)))]
    sizes = [len(b["atom_ptr"]) - 1 for b in subs]
    osub, osam = pk.build_epoch_index(pk.temperature_counts(sizes, 2.0), sizes, seed=5)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    pool = pk.select(pk.concat(subs), offs[osub] + osam)
    G, B = 8, 32
    sched = pk.plan(np.diff(pool["atom_ptr"]), G, B, 4, seed=3, mode="balanced")
    batch = pk.select(pool, sched["sample"][:G * B])
    assert batch["denoise"].sum() > 20 and np.diff(batch["atom_ptr"]).min() >= 8
    D = cases.CFG[4]
    table = cases.random_table(D, seed=8, elements=(8, 14))
    params = oracle_port.init_params(cases.CFG, 3)
    v0 = np.zeros_like(params)
    tc = pk.TrainConfig(seed=19, clip_norm=1e9)
    with oracle_port.periodic(batch["cell"]):
        ref = oracle_port.train_step(cases.CFG, G, B, batch, table, params, v0, seed=tc.seed, step=2,
                                     clip=tc.clip_norm)
    mcfg = pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=D)
    dev = pk.Device(mcfg, seed=0)
    dev.set_params(params)
    dev.set_rms_state(v0)
    dev.set_reference_table(table)
    res = dev.train_step_workers([pk.select(batch, np.arange(g * B, (g + 1) * B)) for g in range(G)], tc, step=2)
    _check_step(res, dev.grads() / G, dev.rms_state(), ref, cases.CFG, "cfg3 periodic G=8 B=32")
    dev.close()


def test_long_pipelined_runs_stay_bit_identical(pk):
    """Soak: 400 headline steps (side-stream prefetch of the next slot, batch-state
    parity swaps) against 400 unpipelined steps, and 300 public pipelined
    submit / wait steps against 300 synchronous train_step calls: every loss and the
    final parameters bit-identical (the loss falls from 8.7 to 0.6 on the way)."""
    import bench
    from paper_2505_22208_b200.dist import shard
    pool, table, sched = bench.make_workload(pk, 1)
    n = sched["n_batches"]
    shards = [shard(pool, sched, s, 0, 1, bench.BATCH_PER_GPU) for s in range(n)]
    cfg = pk.ModelConfig(**bench.CFG)
    tc = pk.TrainConfig(seed=11)

    def staged(pipelined, K=400):
        dev = pk.Device(cfg, seed=7)
        dev.set_reference_table(table)
        for s, b in enumerate(shards):
            dev.stage(b, tc, step=s, slot=s)
        losses = [dev.train_step_staged(k % n, sync=True, next_slot=((k + 1) % n) if pipelined else None).loss
                  for k in range(K)]
        p = dev.params()
        dev.close()
        return losses, p

    def public(pipelined, K=300):
        dev = pk.Device(cfg, seed=7)
        dev.set_reference_table(table)
        if pipelined:
            losses, pending = [], None
            for k in range(K):
                t = dev.train_step_submit(shards[k % n], tc, step=k)
                if pending is not None:
                    losses.append(dev.train_step_wait(pending).loss)
                pending = t
            losses.append(dev.train_step_wait(pending).loss)
        else:
            losses = [dev.train_step(shards[k % n], tc, step=k).loss for k in range(K)]
        p = dev.params()
        dev.close()
        return losses, p

    for run in (staged, public):
        (la, pa), (lb, pb) = run(True), run(False)
        assert la == lb, run.__name__
        assert np.array_equal(pa.view(np.uint64), pb.view(np.uint64)), run.__name__


def test_cfg2_evaluation_at_bench_scale(pk, oracle_ref):
    """The validation path (lamm_evaluate, S/trainer.cpp:528-553) on the heaviest
    cfg2 mini-batch of the bench's epoch (256 molecules, ~14 k atoms, ~300 k edges:
    several TMA chunks per group): physical-unit energy and force MAEs vs the reference."""
    import bench
    from paper_2505_22208_b200.dist import shard
    pool, table, sched = bench.make_workload(pk, 1)
    shards = [shard(pool, sched, s, 0, 1, bench.BATCH_PER_GPU) for s in range(sched["n_batches"])]
    b = max(shards, key=lambda x: int(x["atom_ptr"][-1]))
    b = dict(b)
    b["denoise"] = np.zeros_like(b["denoise"])
    cfg = (bench.CFG["hidden"], bench.CFG["layers"], bench.CFG["rbf"], bench.CFG["cutoff"], bench.CFG["heads"])
    params = oracle_ref.init_params(cfg, 17)
    dev = pk.Device(pk.ModelConfig(**bench.CFG), seed=0)
    dev.set_params(params)
    dev.set_reference_table(table)
    got = dev.evaluate(b)
    dev.close()
    want = oracle_ref.evaluate(cfg, params, b, table)
    assert got["energy_count"] == want["energy_count"] and got["force_count"] == want["force_count"]
    for k in ("energy_mae", "force_mae"):
        assert abs(got[k] - want[k]) <= TOL * abs(want[k]), (k, got[k], want[k])


def test_cfg2_neighbor_lists_bit_exact_at_bench_scale(pk, oracle_ref):
    """Every mini-batch of the bench's cfg2 epoch (256 molecules each, 3-14 k atoms):
    pair set, order, fp64 distances and unit vectors bit-identical to the reference's
    build_neighbor_list (S/core.cpp:30-48), sample by sample."""
    import bench
    from paper_2505_22208_b200.dist import shard
    from test_gpu_parity import check_nlist
    pool, table, sched = bench.make_workload(pk, 1)
    dev = pk.Device(pk.ModelConfig(**bench.CFG), seed=0)
    dev.set_option("export_fp64", 1)
    for s in range(sched["n_batches"]):
        check_nlist(dev, oracle_ref, shard(pool, sched, s, 0, 1, bench.BATCH_PER_GPU))
    dev.close()
