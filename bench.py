#!/usr/bin/env python3
"""Throughput of the load-balanced LaMM energy/force train step on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "cfg2"): per rank a device-batch of 256
synthetic organic molecules (reference generator, lognormal mode 20 sigma 0.5,
5-60 atoms, elements H/C/N/O, Morse labels), model ModelConfig{hidden 128,
layers 3, rbf 16, cutoff 5 A, heads 10} (the reference's model family at the
north star's PaiNN size), scheduled by the balanced plan (G = N workers, B = 256,
S = 16). One step = denoise/normalize -> neighbour list -> forward -> Eq.(5)
loss -> backward -> NCCL allreduce (N > 1) -> clip -> RMS update.

value  : atoms/s over all ranks with inputs resident in HBM (staged slots),
         device time (CUDA events around each step, L2 flushed between steps,
         max over ranks).
e2e    : same metric through the public API (pipelined lamm_train_step_submit/_wait) with host
         batches: host packing, H2D, the step, D2H of the result, per step.
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "atoms/sec per train step"
CFG = dict(hidden=128, layers=3, rbf=16, cutoff=5.0, heads=10)
BATCH_PER_GPU = 256
EPOCH_STEPS = 8
SPLITS = 16
GEN = dict(mode=20.0, sigma=0.5, min_atoms=5, max_atoms=60, elements=(1, 6, 7, 8))
L2_FLUSH = 256 << 20
E2E_FLUSH = 128 << 20  # e2e: larger than the 126 MB (120 MiB) L2, and inside the timed region


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ------------------------------------------------------------ workload
def make_workload(pk, world: int, seed: int = 42):
    """The pool, its reference table and the balanced schedule (identical on all ranks)."""
    pool_n = BATCH_PER_GPU * world * EPOCH_STEPS
    pool = pk.synth_generate(pool_n, seed, threads=os.cpu_count() or 8, **GEN)
    atoms = np.diff(pool["atom_ptr"])
    sched = pk.plan(atoms, world, BATCH_PER_GPU, SPLITS, seed=7, mode="balanced")
    return pool, fit_table(pool, CFG["heads"]), sched


def fit_table(pool, D):
    """Setup-only stand-in for fit_normalizer (S/loss.cpp:64-111): least-squares
    per-element reference energies, residual mean/std, force std; head 0."""
    ap, Z = pool["atom_ptr"], pool["Z"]
    B = len(ap) - 1
    comp = np.zeros((B, 119))
    np.add.at(comp, (np.repeat(np.arange(B), np.diff(ap)), Z), 1.0)
    cols = np.nonzero(comp.sum(0))[0]
    rho_c, *_ = np.linalg.lstsq(comp[:, cols], pool["energy"], rcond=None)
    t = dict(rho=np.zeros((D, 119)), rho_has=np.zeros((D, 119), np.uint8), mean=np.zeros(D), std=np.ones(D),
             fstd=np.ones(D), has=np.ones(D, np.uint8))
    t["rho"][0, cols] = rho_c
    t["rho_has"][0, cols] = 1
    resid = pool["energy"] - comp[:, cols] @ rho_c
    t["mean"][0] = resid.mean()
    t["std"][0] = max(resid.std(), 1e-8)
    t["fstd"][0] = max(pool["forces"].std(), 1e-8)
    return t


# ------------------------------------------------------------ clocks
class ClockSampler:
    """NVML poll (about every 2 ms) of SM clock and clock-event reasons from a
    thread; start() returns once the first sample is in, so the samples cover
    the timed region that follows."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, local_rank: int):
        self.rows, self.max_mhz, self.err = [], None, None
        self._stop = threading.Event()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v for v in vis.split(",") if v.strip()]
        self.index = int(ids[local_rank]) if ids and ids[local_rank].strip().isdigit() else local_rank

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.masks = [(n, getattr(nv, m)) for n, m in self.REASONS]
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            t0 = time.perf_counter()
            while not self.rows and time.perf_counter() - t0 < 2.0:
                time.sleep(0.001)
        except Exception as e:  # no NVML: report unsampled
            self.err = repr(e)
        return self

    def _poll(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((float(sm), int(rs)))
            except Exception as e:
                self.err = repr(e)
                return
            time.sleep(0.002)

    def stop(self):
        self._stop.set()
        if getattr(self, "thread", None):
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "error": self.err}
        reasons = sorted({n for _, rs in self.rows for n, m in self.masks if rs & m})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_min_mhz": min(r[0] for r in self.rows),
                "sm_max_mhz": self.max_mhz, "samples": len(self.rows), "reasons": reasons, "source": "nvml"}


# ------------------------------------------------------------ roofline
def kernel_bytes(name, N, P, H=128, K=16, D=10):
    """Algorithmic bytes per launch, SURVEY.md §8(d)'s model verbatim: fp32
    storage, gather-inclusive (every edge pays its source-row read):
      message   P (4 + 4 + 4H) + N 8H          bwd_edge  P (8 + 8H) + N 12H
                (fused with the update GEMM at H = 128: + N 16H + 4H^2)
      force     P (20 + 4H) + N (4H + 12D)     head_bwd  P (20 + 4H + 12D) + N (8H + 12D)
    (node GEMMs: activations in + out + weights)."""
    e = {
        # k_message_update (H = 128) also runs the layer's update GEMM: + its activations
        # (mu in, h in, h and t out) and W_u
        "message": P * (4 + 4 + 4 * H) + N * 8 * H + N * 16 * H + 4 * H * H,
        "bwd_edge": P * (8 + 8 * H) + N * 12 * H,
        "force": P * (20 + 4 * H) + N * (4 * H + 12 * D),
        "head_bwd": P * (20 + 4 * H + 12 * D) + N * (8 * H + 12 * D),
        "update": N * (4 * H + 4 * H + 8 * H) + 4 * H * H,
        "bwd_gemm": N * (8 * H + 4 * H) + 4 * H * H,
    }
    return e.get(name)


def kernel_bytes_unique(name, N, P, H=128, K=16, D=10):
    """Compulsory (unique) bytes per launch: every array the kernel touches read or
    written once (per-edge metadata as stored: col, dst, {r, fcut}, segment bits;
    per-atom rows once). The gap to the gather-inclusive bytes is L1/L2 reuse of
    the gathered source rows."""
    e = {
        "message": P * (4 + 4 + 8 + 0.125) + N * (4 * H + 4 * H + 4) + N * 16 * H + 4 * H * H,
        "bwd_edge": P * (4 + 4 + 8 + 0.125) + N * (4 * H + 4 * H + 8 * H + 4),
        "force": P * (4 + 4 + 16 + 8 + 0.125) + N * (4 * H + 4 * (3 * H + 3 + 3 * K) + 4),
        "head_bwd": P * (4 + 4 + 8 + 8 + 0.125) + N * (4 * H + 4 * H + 4 * H + 16 + 4),
        "update": N * (4 * H + 4 * H + 8 * H) + 4 * H * H,
        "bwd_gemm": N * (8 * H + 4 * H) + 4 * H * H,
    }
    return e.get(name)


TRAFFIC_JSON = "r02_ncu_traffic.json"


def ncu_traffic(name, algorithmic_bytes, which="cfg2"):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    kernel from the committed ncu --set full capture (profiles/r02_ncu_traffic.json,
    section `which`), scaled from the captured step to this workload by the
    algorithmic bytes."""
    try:
        with open(os.path.join(ROOT, "profiles", TRAFFIC_JSON)) as f:
            k = json.load(f)[which]["kernels"][name]
        return k["dram_bytes"] / k["algorithmic_bytes"] * algorithmic_bytes
    except Exception:
        return None


def kernel_flops(name, N, P, H=128, K=16, D=10):
    return {"update": 2 * N * H * H, "bwd_gemm": 4 * N * H * H, "message": P * (2 * H * K + 3 * H),
            "bwd_edge": P * (4 * H * K + 6 * H)}.get(name)


# ------------------------------------------------------------ arms
def run_ours(args, dist):
    import paper_2505_22208_b200 as pk
    from paper_2505_22208_b200.dist import shard

    if dist.world > 1:
        os.environ.setdefault("CUDA_VISIBLE_DEVICES", os.environ.get("CUDA_VISIBLE_DEVICES", ""))
    gpu = dist.local_rank
    pool, table, sched = make_workload(pk, dist.world)
    mcfg = pk.ModelConfig(**CFG)
    dev = pk.Device(mcfg, device=gpu, seed=7)
    if dist.world > 1:
        # NCCL's INIT lines on stderr (nranks / rank / device of every communicator)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        uid = dist.bcast_bytes(pk.comm_unique_id() if dist.rank == 0 else None)
        dev.comm_init(dist.world, dist.rank, uid)
    dev.set_reference_table(table)
    tc = pk.TrainConfig(seed=11)
    n_steps = sched["n_batches"]
    shards = [shard(pool, sched, s, dist.rank, dist.world, BATCH_PER_GPU) for s in range(n_steps)]
    for s, b in enumerate(shards):
        dev.stage(b, tc, step=s, slot=s, workers=dist.world, rank=dist.rank)
    # warm-up: every slot once (grows all capacities, captures the graphs), then W more;
    # each step also builds the next step's batch preparation (denoise, labels,
    # neighbour list) on a side stream during its model (lamm_train_step_staged_next)
    for k in range(max(args.warmup, 0) + n_steps):
        dev.train_step_staged(k % n_steps, sync=True, next_slot=(k + 1) % n_steps)
    anomalies0 = dev.anomalies()
    K = args.steps

    slot_atoms = [int(b["atom_ptr"][-1]) for b in shards]

    def timed_region(pipelined=True, per_step_sync=True):
        """K steps, each bracketed by CUDA events on the ctx stream inside the
        library (upload -> step -> allreduce -> optimizer, and the next step's batch
        preparation it overlaps); the L2 flush and the result read-back sit outside
        the brackets (every step's result is read before the next, like the
        reference's per-step loss check). Returns (device ms, atoms)."""
        dev.kernel_times_reset()  # also resets the step-time accumulator
        atoms = 0
        comp.clear()
        dist.barrier()
        dev.sync()
        for k in range(K):
            dev.flush_l2(L2_FLUSH)
            dev.train_step_staged(k % n_steps, sync=per_step_sync,
                                  next_slot=(k + 1) % n_steps if pipelined else None)
            atoms += slot_atoms[k % n_steps]
            if per_step_sync and dist.world > 1:  # this rank's upload -> allreduce time (its own work)
                comp.append(dev.last_step_compute_ms())
        dev.sync()
        dist.barrier()
        ms, nsteps = dev.step_times()
        assert nsteps == K, (nsteps, K)
        return ms, atoms

    # ---- timed region (device-resident inputs, no per-kernel events)
    comp = []
    clk = ClockSampler(gpu).start()
    dev_ms, atoms_local = timed_region()
    clk.stop()
    live_imb = None
    if dist.world > 1:  # the north star's max/mean per-rank step time, from the concurrent ranks themselves
        c = np.asarray(comp, np.float64)
        cmax, csum = dist.allreduce_array(c, "max"), dist.allreduce_array(c, "sum")
        r = cmax / (csum / dist.world)
        live_imb = {"time_mean": float(r.mean()), "time_p95": float(np.percentile(r, 95)), "steps": int(len(r)),
                    "per_rank_time": "device time from the step's upload to its gradient allreduce (event inside "
                                     "the step graph), each rank; max / mean over ranks per step"}
    launches = dev.last_step_launches() * K
    ms_max = dist.allreduce(dev_ms, "max")
    atoms_all = dist.allreduce(float(atoms_local), "sum")
    value = atoms_all / (ms_max / 1e3)
    # ---- the same K steps again with an event pair around every kernel (the
    # graph is re-captured with event-record nodes): per-kernel durations
    dev.set_option("profile", 1)
    dev.train_step_staged(0, sync=True)
    prof_ms, _ = timed_region(pipelined=False)
    ktimes = dev.kernel_times()
    dev.set_option("profile", 0)
    assert dev.anomalies() == anomalies0, "a timed step skipped its update (capacity overflow or non-finite)"
    # per-step edges for the roofline (one synced pass over the slots)
    edge_counts = []
    for s in range(n_steps):
        r = dev.train_step_staged(s, sync=True)
        edge_counts.append(r.n_edges)
    # ---- e2e: public API with host batches, pipelined (lamm_train_step_submit /
    # lamm_train_step_wait: the host packs step k+1 while the device runs step k).
    # Every step's H2D of its packed batch and D2H of its result header are inside
    # the wall-clock region, and so is the L2 flush enqueued between steps.
    def e2e_pass(n):
        h2d = d2h = atoms = 0
        pending = None
        for k in range(n):
            s = k % n_steps
            t = dev.train_step_submit(shards[s], tc, step=s, workers=dist.world, rank=dist.rank)
            dev.flush_l2(E2E_FLUSH)
            if pending is not None:
                r = dev.train_step_wait(pending)
                h2d, d2h, atoms = h2d + r.h2d_bytes, d2h + r.d2h_bytes, atoms + r.n_atoms
            pending = t
        r = dev.train_step_wait(pending)
        return h2d + r.h2d_bytes, d2h + r.d2h_bytes, atoms + r.n_atoms

    e2e_pass(max(args.warmup, 3))
    dist.barrier()
    dev.sync()
    t0 = time.perf_counter()
    h2d, d2h, e2e_atoms = e2e_pass(K)
    e2e_s = time.perf_counter() - t0
    e2e_max = dist.allreduce(e2e_s, "max")
    e2e_atoms_all = dist.allreduce(float(e2e_atoms), "sum")
    e2e = e2e_atoms_all / e2e_max
    # ---- roofline of the dominant kernel
    hbm, tflops, src = peaks()
    steps_done = K
    N_mean = atoms_local / K
    P_mean = float(np.mean([edge_counts[k % n_steps] for k in range(K)]))
    edges_all = dist.allreduce(float(sum(edge_counts[k % n_steps] for k in range(K))), "sum")
    tot_ms = sum(v[0] for v in ktimes.values())
    top = max(ktimes.items(), key=lambda kv: kv[1][0]) if ktimes else ("none", (0.0, 1))
    tname, (tms, tcount) = top
    per_launch_ms = tms / max(tcount, 1)
    launches_per_step = tcount / steps_done
    byts = kernel_bytes(tname, N_mean, P_mean)
    roof = {"kernel": tname, "bound": "hbm", "unit": "GB/s", "peak": hbm, "peak_source": src,
            "bytes_model": "SURVEY.md §8(d) (gather-inclusive, fp32 storage)",
            "traffic_source": f"profiles/{TRAFFIC_JSON} (ncu --set full, DRAM bytes / algorithmic bytes of the "
                              "captured cfg2 step, times this workload's algorithmic bytes)",
            "share_of_step": tms / tot_ms if tot_ms else None, "avg_launch_us": per_launch_ms * 1e3,
            "launches_per_step": launches_per_step,
            "timing": "CUDA event pair around each launch on the ctx stream, second pass over the same K steps "
                      "(profiled step %.3f ms vs %.3f ms unprofiled)" % (prof_ms / K, dev_ms / K)}
    if byts is not None:
        ach = byts / (per_launch_ms / 1e3) / 1e9
        ub = kernel_bytes_unique(tname, N_mean, P_mean)
        roof.update(achieved=ach, frac=ach / hbm, traffic=ncu_traffic(tname, byts), algorithmic_bytes_per_launch=byts,
                    compulsory_bytes_per_launch=ub, compulsory_frac=ub / (per_launch_ms / 1e3) / 1e9 / hbm)
    fl = kernel_flops(tname, N_mean, P_mean)
    if fl is not None:
        roof["fp32_flops_per_launch"] = fl
    kern = {k: {"ms_per_step": v[0] / steps_done, "launches_per_step": v[1] / steps_done,
                "share": v[0] / tot_ms if tot_ms else None} for k, v in sorted(ktimes.items(), key=lambda kv: -kv[1][0])}
    out = {
        "metric": METRIC, "value": value, "unit": "atoms/s", "n_gpus": dist.world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
        "edges_per_s": edges_all / (ms_max / 1e3),
        "vs_baseline": None, "dtype": "f32 (fp64 neighbour list/optimizer)", "data": "synthetic",
        "config": {"workload": "cfg2: mixed organic molecules 5-60 atoms, batch 256 per GPU, non-periodic",
                   "model": "LaMM MPNN hidden128 layers3 rbf16 cutoff5 heads10 (74,400 params)",
                   "global_batch": BATCH_PER_GPU * dist.world, "atoms_per_step_per_gpu": N_mean,
                   "edges_per_step_per_gpu": P_mean, "parallelism": f"dp{dist.world}",
                   "schedule": "balanced (G=%d, B=%d, S=%d)" % (dist.world, BATCH_PER_GPU, SPLITS),
                   "l2": "flushed between timed steps (256 MiB memset outside the events)",
                   "inputs": "value: device-resident staged batches; e2e: host batches via lamm_train_step_submit/_wait"},
        "e2e": {"value": e2e, "unit": "atoms/s", "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
                "ms_per_step": e2e_max / K * 1e3,
                "method": "wall clock over K pipelined lamm_train_step_submit/_wait calls with host batches "
                          "(pack + H2D + step + D2H of the result per step; a 128 MiB L2 flush (> the 126 MB L2) "
                          "between steps is inside the timed region)"},
        "gpu_launches": launches,
        "roofline": roof,
        "rank_imbalance_live": live_imb,
        "kernels": kern,
        "clocks": clk.summary(),
    }
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(budget_s=args.cpu_budget)
    if dist.rank == 0 and dist.world == 1 and not args.no_imbalance:
        out["rank_imbalance"] = rank_imbalance(pk, dev, pool, table, tc)
        out["rank_imbalance_heavy_tail"] = rank_imbalance_heavy(pk, dev, tc)
        out["periodic_cfg1"] = periodic_cfg1(pk, mcfg, tc)
        out["semisup_cfg3"] = semisup_cfg3(pk, mcfg, tc)
        out["semisup_cfg3_periodic"] = semisup_cfg3(pk, mcfg, tc, periodic=True)
        out["cost_balancing"] = cost_balancing(pk, mcfg, tc)
        out["batch_sweep"] = batch_sweep(pk, mcfg, tc)
        out["supercells_cfg4"] = supercells_cfg4(pk, mcfg, tc)
    if dist.rank == 0 and dist.world == 1 and not args.no_large:
        out["roofline_large"] = roofline_large(pk, mcfg, tc)
    dev.close()
    return out


def np_select(batch: dict, ids) -> dict:
    """Plain-numpy sample selection (the reference arm must not import the product)."""
    ap = batch["atom_ptr"]
    ids = np.asarray(ids, np.int64)
    sizes = ap[ids + 1] - ap[ids]
    nap = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    rows = np.concatenate([np.arange(ap[i], ap[i + 1]) for i in ids])
    out = dict(atom_ptr=nap)
    for k in ("pos", "Z", "forces"):
        out[k] = np.ascontiguousarray(batch[k][rows])
    for k in ("dataset_index", "energy_mask", "force_mask", "energy", "denoise"):
        out[k] = np.ascontiguousarray(batch[k][ids])
    return out


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "affinity_cores": len(os.sched_getaffinity(0)), "cpu_model": model}


def time_reference_steps(lib, batches, table, cfg, threads, reps, pin_core=None):
    """The reference's own step body (oracle/_ref lref_train_step = S/trainer.cpp:258-327
    on lamm_ref:: calls; threads = 1: the faithful sequential run_loop, > 1: its
    parallel_for over samples) over full device-batches; parameters and RMS state
    carried from step to step. pin_core: taskset-like affinity for the run.
    Returns (per-step seconds, atoms per step)."""
    params = lib.init_params(cfg, 7)
    v = np.zeros_like(params)
    old = os.sched_getaffinity(0)
    if pin_core is not None:
        os.sched_setaffinity(0, {pin_core})
    try:
        secs, atoms = [], []
        for k in range(reps):
            b = batches[k % len(batches)]
            kw = dict(threads=threads) if lib.kind == "ref" else {}
            t0 = time.perf_counter()
            r = lib.train_step(cfg, 1, len(b["atom_ptr"]) - 1, b, table, params, v, seed=11, step=k, **kw)
            secs.append(time.perf_counter() - t0)
            atoms.append(int(b["atom_ptr"][-1]))
            params, v = r["params"], r["rms_v"]
    finally:
        os.sched_setaffinity(0, old)
    return secs, atoms


def reference_workload():
    """cfg2 exactly as make_workload builds it, from the reference's own generator,
    planner and plain numpy (no product code)."""
    import oracle
    lib = oracle.ref() if oracle.ref_available() else oracle.port()
    pool = lib.synth_generate(BATCH_PER_GPU * EPOCH_STEPS, 42, **GEN)
    sched = lib.plan(np.diff(pool["atom_ptr"]), 1, BATCH_PER_GPU, SPLITS, 7, mode="balanced")
    batches = [np_select(pool, sched["sample"][s * BATCH_PER_GPU:(s + 1) * BATCH_PER_GPU])
               for s in range(sched["n_batches"])]
    cfg = tuple(CFG[k] for k in ("hidden", "layers", "rbf", "cutoff", "heads"))
    return lib, batches, fit_table(pool, CFG["heads"]), cfg


def cpu_baseline(budget_s=20.0):
    """The reference's own step (oracle/_ref) on this box's host cores over FULL
    256-molecule cfg2 device-batches: all host threads (median of >= 5 steps) and one
    core (taskset to core 0, threads = 1, the faithful sequential loop)."""
    lib, batches, table, cfg = reference_workload()
    threads = len(os.sched_getaffinity(0))
    time_reference_steps(lib, batches, table, cfg, threads, 1)  # warm-up (page-in, thread pool)
    secs, atoms = time_reference_steps(lib, batches, table, cfg, threads, 5)
    while sum(secs) < budget_s * 0.5 and len(secs) < 40:
        s2, a2 = time_reference_steps(lib, batches, table, cfg, threads, 5)
        secs, atoms = secs + s2, atoms + a2
    med = float(np.median([a / s for a, s in zip(atoms, secs)]))
    s1, a1 = time_reference_steps(lib, batches, table, cfg, 1, 1, pin_core=sorted(os.sched_getaffinity(0))[0])
    kind = "reference" if lib.kind == "ref" else "port"
    return {"value": med, "unit": "atoms/s", "cores": threads if kind == "reference" else 1, "kind": kind,
            "sample": f"median over {len(secs)} full cfg2 steps (256 molecules, {int(np.mean(atoms))} atoms mean), "
                      f"oracle/_ref lref_train_step (S/trainer.cpp:258-327) with {threads} threads",
            "one_core": {"value": a1[0] / s1[0], "unit": "atoms/s", "cores": 1,
                         "sample": f"1 full cfg2 step ({a1[0]} atoms), taskset core 0, threads 1 "
                                   "(the reference's sequential run_loop)"},
            **cpu_info()}


def rank_imbalance(pk, dev, pool, table, tc, G=8, steps=8):
    """Per-rank step time on the one GPU: each of G ranks' shards timed as its own
    device-batch (B = 256/G) for the balanced and naive plans; max/mean per step."""
    out = {"G": G, "batch_per_rank": BATCH_PER_GPU // G}
    dev.set_option("rank_local", 1)  # each rank's share timed on its own (no communicator)
    atoms = np.diff(pool["atom_ptr"])
    for mode in ("balanced", "naive"):
        sched = pk.plan(atoms, G, BATCH_PER_GPU // G, SPLITS, seed=7, mode=mode)
        ratios, aratios = [], []
        per = BATCH_PER_GPU
        for s in range(min(steps, sched["n_batches"])):
            ids = sched["sample"][s * per:(s + 1) * per]
            times = []
            for g in range(G):
                sub = pk.select(pool, ids[g * (per // G):(g + 1) * (per // G)])
                dev.stage(sub, tc, step=s, slot=900 + g, workers=G, rank=g)
                dev.train_step_staged(900 + g, sync=True)  # warm capacity
                ms = []
                for rep in range(3):
                    dev.event_record(0)
                    dev.train_step_staged(900 + g, sync=False)
                    dev.event_record(1)
                    ms.append(dev.event_elapsed_ms(0, 1))
                times.append(min(ms))
            ratios.append(max(times) / np.mean(times))
            wa = sched["worker_atoms"][s * G:(s + 1) * G]
            aratios.append(wa.max() / wa.mean())
        out[mode] = {"time_mean": float(np.mean(ratios)), "time_p95": float(np.percentile(ratios, 95)),
                     "atoms_mean": float(np.mean(aratios)), "atoms_max": float(np.max(aratios)),
                     "steps": len(ratios)}
    return out


def periodic_cfg1(pk, mcfg, tc, steps=20):
    """BASELINE configs[0] on the GPU: 32 periodic 64-atom bulk cells (2x2x2 diamond
    Si supercells, 0.05 A jitter, minimum image), full train step per batch;
    a separate context so the headline run is untouched."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cases
    parts = []
    for s in range(32):
        pos, Z, cell = cases.diamond_supercell(seed=100 + s)
        n = len(Z)
        parts.append(dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z, forces=np.zeros((n, 3)),
                          dataset_index=np.zeros(1, np.int32), energy_mask=np.ones(1, np.uint8),
                          force_mask=np.ones(1, np.uint8), energy=np.array([-4.6 * n]),
                          denoise=np.zeros(1, np.uint8), cell=cell[None]))
    batch = pk.concat(parts)
    dev = pk.Device(mcfg, seed=7)
    dev.stage(batch, tc, step=0, slot=0)
    for _ in range(3):
        dev.train_step_staged(0, sync=True)
    dev.kernel_times_reset()
    edges = 0
    for _ in range(steps):
        dev.flush_l2(L2_FLUSH)
        edges = dev.train_step_staged(0, sync=True).n_edges
    ms, n = dev.step_times()
    dev.close()
    atoms = int(batch["atom_ptr"][-1])
    return {"workload": "cfg1: 32 periodic 64-atom Si diamond supercells (minimum image), train step",
            "atoms_per_step": atoms, "edges_per_step": edges, "ms_per_step": ms / n, "atoms_per_s": atoms / (ms / n / 1e3)}


def rank_imbalance_heavy(pk, dev, tc, G=8, B=4, S=64, steps=8):
    """cfg5-like load-balancer stress: heavy-tailed sizes (lognormal mode 20,
    sigma 1.0, 2-2000 atoms) scheduled for G ranks x B samples, the per-rank
    device steps timed on this GPU; plus the schedule-only atom imbalance of a
    1M-sample trace at G = 2/4/8 (B = 4, S = 10,000)."""
    out = {"pool": "synthetic clusters, lognormal(mode 20, sigma 1.0), 2-2000 atoms", "G": G, "batch_per_rank": B}
    n_pool = G * B * S
    pool = pk.synth_generate(n_pool, 5, threads=os.cpu_count() or 8, mode=20.0, sigma=1.0, min_atoms=2,
                             max_atoms=2000, elements=(1, 6, 7, 8))
    atoms = np.diff(pool["atom_ptr"])
    out["pool_atoms_mean"], out["pool_atoms_max"] = float(atoms.mean()), int(atoms.max())
    table = fit_table(pool, CFG["heads"])
    dev.set_reference_table(table)
    dev.set_option("rank_local", 1)
    samples = []  # (rank atoms, device ms) for the simulator's cost-model fit
    for mode in ("balanced", "naive"):
        sched = pk.plan(atoms, G, B, 4, seed=7, mode=mode)
        per = G * B
        ratios, aratios, pred = [], [], []
        for s in range(min(steps, sched["n_batches"])):
            ids = sched["sample"][s * per:(s + 1) * per]
            times = []
            for g in range(G):
                sub = pk.select(pool, ids[g * B:(g + 1) * B])
                dev.stage(sub, tc, step=s, slot=950 + g, workers=G, rank=g)
                dev.train_step_staged(950 + g, sync=True, next_slot=950 + g)
                ms = []
                for rep in range(3):
                    dev.event_record(0)
                    dev.train_step_staged(950 + g, sync=False, next_slot=950 + g)
                    dev.event_record(1)
                    ms.append(dev.event_elapsed_ms(0, 1))
                times.append(min(ms))
            ratios.append(max(times) / np.mean(times))
            wa = sched["worker_atoms"][s * G:(s + 1) * G]
            aratios.append(wa.max() / wa.mean())
            samples += list(zip(wa.tolist(), times))
            pred.append(wa)
        out[mode] = {"time_mean": float(np.mean(ratios)), "time_p95": float(np.percentile(ratios, 95)),
                     "atoms_mean": float(np.mean(aratios)), "atoms_max": float(np.max(aratios)),
                     "steps": len(ratios), "_worker_atoms": pred}
    # the reference's step-time simulator (S/simulator.cpp:19-59: per worker
    # alpha + beta * atoms, step = slowest worker) with alpha/beta fitted to these
    # B200 per-rank times: predicted vs measured max/mean per step
    a, t = np.array([x[0] for x in samples], float), np.array([x[1] for x in samples], float)
    beta, alpha = np.polyfit(a, t, 1)
    sim = {"alpha_ms": float(alpha), "beta_us_per_atom": float(beta * 1e3),
           "fit_r2": float(1 - np.sum((t - alpha - beta * a) ** 2) / np.sum((t - t.mean()) ** 2))}
    for mode in ("balanced", "naive"):
        # the native simulator (lamm_simulate, bit-exact with S/simulator.cpp:19-59) on
        # the timed steps' worker atoms with the fitted alpha / beta (one GPU: gamma,
        # delta = 0): per step the slowest worker and the summed idle give max / mean
        wa = np.concatenate(out[mode].pop("_worker_atoms"))
        nb = len(wa) // G
        sr = pk.simulate({"n_batches": nb, "worker_atoms": wa, "sample": np.zeros(nb * G * B, np.int64)},
                         alpha_s=max(alpha, 0.0) * 1e-3, beta_s_per_atom=max(beta, 1e-12) * 1e-3, gamma_s=0.0,
                         delta_s=0.0)
        slow = sr["step_time"]
        p = slow / (slow - sr["step_idle"] / G)
        sim[mode] = {"predicted_time_mean": float(np.mean(p)), "measured_time_mean": out[mode]["time_mean"],
                     "predicted_by": "lamm_simulate"}
    out["simulator_cross_check"] = sim
    trace = pk.make_trace("lognormal", count=1_000_000, min_atoms=2, max_atoms=2000, mode=20.0, sigma=1.0, seed=3)
    sched_1m = {}
    for g in (2, 4, 8):
        row = {}
        for mode in ("balanced", "naive"):
            sc = pk.plan(trace, g, 4, 10_000, seed=3, mode=mode)
            row[mode] = {"mean_imbalance": sc["mean_imbalance"], "max_imbalance": sc["max_imbalance"],
                         "steps": sc["n_batches"], "dropped": sc["dropped"]}
        sched_1m[f"G{g}"] = row
    out["schedule_1M_trace_atoms"] = sched_1m
    return out


def pair_counts(pk, dev, pool, chunk=512):
    """Directed pair count per sample, from the device neighbour list (bit-exact
    with the reference's build_neighbor_list), chunk samples at a time."""
    B = len(pool["atom_ptr"]) - 1
    out = np.zeros(B, np.int64)
    for s0 in range(0, B, chunk):
        sub = pk.select(pool, np.arange(s0, min(B, s0 + chunk)))
        dev.set_batch(sub)
        ptr = dev.build_neighbor_list(fp64=False)[0]
        out[s0:s0 + len(ptr) - 1] = np.diff(ptr)
    return out


def cost_balancing(pk, mcfg, tc, G=8, B=48, steps=6):
    """North star: "assigns samples to ranks by predicted atom/edge cost". A mixed
    pool where atoms alone mispredict the work: cfg2-like molecules (~17 pairs per
    atom), periodic crystals (~40, with images) and Si supercells (28). (1) the
    reference's atom-balanced plan, every rank slice timed; (2) the step-time model
    t = t0 + per_atom * atoms + per_edge * edges fitted to those times
    (pk.fit_cost_model); (3) a fresh schedule seed planned by atoms and by the
    fitted cost (lamm_plan_cost), both timed: max/mean per-rank time per step."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cases
    rng = np.random.default_rng(17)
    mol = pk.synth_generate(2400, 31, threads=os.cpu_count() or 8, mode=30.0, sigma=0.6, min_atoms=5, max_atoms=200,
                            elements=(1, 6, 7, 8))
    mol["denoise"] = np.zeros(len(mol["atom_ptr"]) - 1, np.uint8)
    cry = crystal_pool(pk, 1000, 33, "energy_and_forces", 40.0, sigma=0.6)
    sc = []
    for k in range(200):
        pos, Z, cell = cases.diamond_supercell(reps=tuple(rng.integers(2, 4, 3)), seed=3000 + k)
        n = len(Z)
        sc.append(dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z, forces=rng.normal(0, 0.1, (n, 3)),
                       dataset_index=np.zeros(1, np.int32), energy_mask=np.ones(1, np.uint8),
                       force_mask=np.ones(1, np.uint8), energy=np.array([-4.6 * n]), denoise=np.zeros(1, np.uint8),
                       cell=cell[None]))
    pool = pk.concat([mol, cry] + sc)
    pool = pk.select(pool, rng.permutation(len(pool["atom_ptr"]) - 1))
    atoms = np.diff(pool["atom_ptr"])
    dev = pk.Device(mcfg, seed=7)
    edges = pair_counts(pk, dev, pool)
    dev.set_option("rank_local", 1)
    dev.set_reference_table(fit_table(mol, CFG["heads"]))

    def timed(sched):
        rows = time_rank_slices(pk, dev, pool, sched, G, B, tc, steps, slot0=900)
        per = G * B
        a, e, t, r = [], [], [], []
        for s, (ra, rt) in enumerate(rows):
            ids = sched["sample"][s * per:(s + 1) * per]
            re = [int(edges[ids[g * B:(g + 1) * B]].sum()) for g in range(G)]
            a += ra.tolist()
            e += re
            t += rt.tolist()
            r.append(rt.max() / rt.mean())
        return a, e, t, r

    fa, fe, ft, fr = timed(pk.plan(atoms, G, B, 8, seed=5, mode="balanced"))
    cm, t0, r2 = pk.fit_cost_model(fa, fe, ft)
    _, _, _, ra = timed(pk.plan(atoms, G, B, 8, seed=6, mode="balanced"))
    pc = pk.plan_cost(atoms, edges, cm, G, B, 8, seed=6, mode="balanced")
    _, _, _, rc = timed(pc)
    return {"pool": "2400 molecules (5-200 atoms) + 1000 periodic crystals (8-200) + 200 Si supercells (64-216), "
                    "shuffled", "G": G, "batch_per_rank": B, "pool_atoms_mean": float(atoms.mean()),
            "pool_edges_per_atom": float(edges.sum() / atoms.sum()),
            "fit": {"t0_ms": t0, "per_atom_us": cm.per_atom * 1e3, "per_edge_us": cm.per_edge * 1e3, "r2": r2,
                    "on": f"{len(ft)} rank steps of the atom-balanced plan, schedule seed 5"},
            "atoms_balanced": {"time_imbalance_mean": float(np.mean(ra)), "time_imbalance_p95": float(np.percentile(ra, 95)),
                               "steps": len(ra)},
            "cost_balanced": {"time_imbalance_mean": float(np.mean(rc)), "time_imbalance_p95": float(np.percentile(rc, 95)),
                              "predicted_cost_imbalance_mean": pc["cost_imbalance_mean"], "steps": len(rc)},
            "evaluated_on": "schedule seed 6 (not the fit's)"}


def time_rank_slices(pk, dev, pool, sched, G, B, tc, steps, slot0=970):
    """Per scheduled mini-batch, each of the G ranks' B-sample slices staged and
    timed as its own device step on this GPU (min of 3, CUDA events on the ctx
    stream; the next step's batch preparation built during each step, as in the
    headline loop); returns [(rank atoms [G], rank ms [G])] per step."""
    out = []
    per = G * B
    for s in range(min(steps, sched["n_batches"])):
        ids = sched["sample"][s * per:(s + 1) * per]
        atoms, times = [], []
        for g in range(G):
            sub = pk.select(pool, ids[g * B:(g + 1) * B])
            dev.stage(sub, tc, step=s, slot=slot0 + g, workers=G, rank=g)
            dev.train_step_staged(slot0 + g, sync=True, next_slot=slot0 + g)
            ms = []
            for _ in range(3):  # as in the headline loop: the next step's batch preparation overlaps
                dev.event_record(0)
                dev.train_step_staged(slot0 + g, sync=False, next_slot=slot0 + g)
                dev.event_record(1)
                ms.append(dev.event_elapsed_ms(0, 1))
            atoms.append(int(sub["atom_ptr"][-1]))
            times.append(min(ms))
        out.append((np.array(atoms), np.array(times)))
    return out


def slice_summary(rows):
    """max/mean per-rank time per step, and the per-GPU throughput of the slices."""
    r = [t.max() / t.mean() for _, t in rows]
    a = sum(x.sum() for x, _ in rows)
    t = sum(t.sum() for _, t in rows)
    return {"time_imbalance_mean": float(np.mean(r)), "time_imbalance_p95": float(np.percentile(r, 95)),
            "atoms_per_s_per_gpu": float(a / (t / 1e3)), "steps": len(rows)}


def supercells_cfg4(pk, mcfg, tc, Gs=(2, 4, 8), B=4, steps=6):
    """BASELINE configs[3]: periodic diamond-Si supercells of r0 x r1 x r2 cubic cells
    (r in 3..5: 216-1000 atoms, 28 neighbours per atom within 5 A), B = 4 per rank;
    the balanced and naive plans at G = 2/4/8 with every rank's slice timed as a
    full train step on this GPU (per-rank device work; the allreduce is not in
    these times). Also the single-GPU step throughput (G = 1)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cases
    rng = np.random.default_rng(11)
    parts = []
    for s in range(8 * B * steps):
        pos, Z, cell = cases.diamond_supercell(reps=tuple(rng.integers(3, 6, 3)), seed=1000 + s)
        n = len(Z)
        parts.append(dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z,
                          forces=rng.normal(0, 0.1, (n, 3)), dataset_index=np.zeros(1, np.int32),
                          energy_mask=np.ones(1, np.uint8), force_mask=np.ones(1, np.uint8),
                          energy=np.array([-4.6 * n + rng.normal()]), denoise=np.zeros(1, np.uint8),
                          cell=cell[None]))
    pool = pk.concat(parts)
    atoms = np.diff(pool["atom_ptr"])
    dev = pk.Device(mcfg, seed=7)
    dev.set_option("rank_local", 1)
    dev.set_reference_table(fit_table(pool, CFG["heads"]))
    out = {"workload": "cfg4: periodic diamond-Si supercells 216-1000 atoms (3-5 cubic cells per axis), "
                       "B = 4 per rank, minimum image + cell lists",
           "pool_atoms_mean": float(atoms.mean()), "B": B}
    one = time_rank_slices(pk, dev, pool, pk.plan(atoms, 1, B, 4, seed=3, mode="balanced"), 1, B, tc, steps)
    out["G1"] = {"atoms_per_s": slice_summary(one)["atoms_per_s_per_gpu"],
                 "edges_per_atom": 28}
    for G in Gs:
        row = {}
        for mode in ("balanced", "naive"):
            sched = pk.plan(atoms, G, B, 4, seed=3, mode=mode)
            row[mode] = slice_summary(time_rank_slices(pk, dev, pool, sched, G, B, tc, steps))
        out[f"G{G}"] = row
    dev.close()
    return out


LARGE_B = 48  # 1,000-atom supercells per step: N = 48,000, P = 1.344 M (working set >> the 126 MB L2)


def large_batch(pk, B=LARGE_B, reps=5, seed=2000):
    """B periodic diamond-Si supercells of reps^3 cubic cells (1,000 atoms at reps
    5, 28 neighbours each within 5 A), random labels: one device-batch whose
    per-layer features alone (h, t, mu: 3 x N x 512 B) exceed the L2."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cases
    rng = np.random.default_rng(seed)
    parts = []
    for s in range(B):
        pos, Z, cell = cases.diamond_supercell(reps=reps, seed=seed + s)
        n = len(Z)
        parts.append(dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z,
                          forces=rng.normal(0, 0.1, (n, 3)), dataset_index=np.array([s % CFG["heads"]], np.int32),
                          energy_mask=np.ones(1, np.uint8), force_mask=np.ones(1, np.uint8),
                          energy=np.array([-4.6 * n + rng.normal()]), denoise=np.zeros(1, np.uint8),
                          cell=cell[None]))
    return pk.concat(parts)


def roofline_large(pk, mcfg, tc, steps=5):
    """the edge kernels' roofline on a device-batch larger
    than L2 (LARGE_B x 1,000-atom supercells), where the HBM bound is meaningful.
    Per kernel: event-timed launch duration (profiled pass), SURVEY §8(d)
    gather-inclusive bytes and compulsory (unique) bytes as fractions of the
    measured HBM peak, and the ncu DRAM bytes per launch of the committed capture
    (profiles/r02_ncu_traffic.json, section "large") when present."""
    hbm, _, src = peaks()
    batch = large_batch(pk)
    N = int(batch["atom_ptr"][-1])
    dev = pk.Device(mcfg, seed=7)
    dev.set_reference_table(fit_table(batch, CFG["heads"]))
    dev.stage(batch, tc, step=0, slot=0)
    for _ in range(3):
        r = dev.train_step_staged(0, sync=True, next_slot=0)
    P = r.n_edges
    dev.kernel_times_reset()
    for _ in range(steps):  # the next step's batch preparation overlaps each step (as in the headline)
        dev.flush_l2(L2_FLUSH)
        dev.train_step_staged(0, sync=True, next_slot=0)
    tot_ms, nst = dev.step_times()
    ms = [tot_ms / nst]
    dev.set_option("profile", 1)
    dev.train_step_staged(0, sync=True)
    dev.kernel_times_reset()
    for _ in range(steps):
        dev.flush_l2(L2_FLUSH)
        dev.train_step_staged(0, sync=True)
    kt = dev.kernel_times()
    dev.set_option("profile", 0)
    dev.close()
    step_ms = float(np.median(ms))
    kern = {}
    for name in ("bwd_edge", "message", "head_bwd", "force", "update", "bwd_gemm"):
        if name not in kt:
            continue
        tot, cnt = kt[name]
        us = tot / cnt * 1e3
        b8, bu = kernel_bytes(name, N, P), kernel_bytes_unique(name, N, P)
        row = {"launches_per_step": cnt / steps, "avg_launch_us": us,
               "s8d_bytes": b8, "s8d_GBs": b8 / us / 1e3, "s8d_frac": b8 / us / 1e3 / hbm,
               "compulsory_bytes": bu, "compulsory_GBs": bu / us / 1e3, "compulsory_frac": bu / us / 1e3 / hbm,
               "share_of_step": tot / sum(v[0] for v in kt.values())}
        tr = ncu_traffic(name, b8, which="large")
        if tr is not None:
            row["ncu_dram_bytes"] = tr
            row["ncu_dram_over_compulsory"] = tr / bu
        kern[name] = row
    return {"workload": f"{LARGE_B} periodic diamond-Si supercells of 1,000 atoms (5x5x5 cubic cells), one "
                        "device-batch per step, L2 flushed between steps", "atoms": N, "edges": P,
            "ms_per_step": step_ms, "atoms_per_s": N / step_ms * 1e3, "peak_GBs": hbm, "peak_source": src,
            "kernels": kern}


def crystal_pool(pk, count, seed, task, mode, sigma=0.5, lo=8, hi=200, dataset_index=0):
    """Periodic crystals for the literal cfg3: n ~ lognormal(mode, sigma) clamped to
    [lo, hi] atoms on randomly chosen sites of a k^3 simple-cubic grid (k^3 >= n,
    spacing 2.3 A, 0.08 A jitter) in a sheared cell of k * 2.3 A: small crystals
    (4.6-9.2 A cells) need several images per pair, large ones take the minimum
    image and cell lists. Elements Si/O; Morse-like random labels (parity only needs
    them finite); task as the reference's subset tasks."""
    rng = np.random.default_rng(seed)
    mu = np.log(mode) + sigma * sigma
    parts = []
    for _ in range(count):
        n = int(np.clip(np.rint(rng.lognormal(mu, sigma)), lo, hi))
        k = int(np.ceil(n ** (1 / 3) - 1e-9))
        a = 2.3
        sites = rng.choice(k ** 3, n, replace=False)
        grid = np.stack(np.unravel_index(sites, (k, k, k)), 1).astype(float)
        cell = np.eye(3) * k * a
        cell[1, 0] = rng.uniform(-0.2, 0.2) * k * a  # shear: triclinic
        pos = (grid + 0.25) / k @ cell + rng.normal(0, 0.08, (n, 3))
        Z = rng.choice(np.array([8, 14], np.int32), n)
        parts.append(dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z, forces=rng.normal(0, 0.3, (n, 3)),
                          dataset_index=np.array([dataset_index], np.int32),
                          energy_mask=np.array([task != "denoising"], np.uint8),
                          force_mask=np.array([task == "energy_and_forces"], np.uint8),
                          energy=np.array([-5.0 * n + rng.normal()]),
                          denoise=np.array([task == "denoising"], np.uint8), cell=cell[None]))
    return pk.concat(parts)


def batch_sweep(pk, mcfg, tc, sizes=(1, 16, 64, 256, 1024, 4096), steps=10):
    """Throughput against the device-batch size for cfg2's molecules (the same
    generator; one slot per size, pipelined steps, L2 flushed between steps): where
    the fixed per-step cost (~18 kernels' critical paths) stops dominating."""
    dev = pk.Device(mcfg, seed=7)
    out = []
    for n in sizes:
        b = pk.synth_generate(n, 77, threads=os.cpu_count() or 8, **GEN)
        dev.set_reference_table(fit_table(b, CFG["heads"]) if n > 8 else None)
        dev.stage(b, tc, step=0, slot=0)
        for _ in range(3):
            r = dev.train_step_staged(0, sync=True, next_slot=0)
        dev.kernel_times_reset()
        for _ in range(steps):
            dev.flush_l2(L2_FLUSH)
            dev.train_step_staged(0, sync=True, next_slot=0)
        ms, k = dev.step_times()
        out.append({"molecules": n, "atoms": r.n_atoms, "edges": r.n_edges, "ms_per_step": ms / k,
                    "atoms_per_s": r.n_atoms / (ms / k) * 1e3})
    dev.close()
    return out


def semisup_cfg3(pk, mcfg, tc, G=8, B=32, steps=6, periodic=False):
    """BASELINE configs[2] (non-periodic twin): three subsets of
    reference-generator structures clamped to 8-200 atoms — E+F labeled (mode 15),
    energy-only (mode 60), coordinate-denoising (mode 30, sigma 0.3 A, centered) —
    mixed at temperature T = 2 into the epoch index, one head per subset, the
    balanced (and naive) plan at G = 8, B = 32; every rank's slice timed as a full
    train step on this GPU."""
    subs = []
    for k, (task, mode, n) in enumerate((("energy_and_forces", 15.0, 3000), ("energy_only", 60.0, 600),
                                         ("denoising", 30.0, 1500))):
        if periodic:
            b = crystal_pool(pk, n, 21 + k, task, mode, dataset_index=k)
        else:
            b = pk.synth_generate(n, 21 + k, task=task, mode=mode, sigma=0.5, min_atoms=8, max_atoms=200,
                                  elements=(1, 6, 7, 8), threads=os.cpu_count() or 8, dataset_index=k)
        subs.append(b)
    sizes = [len(b["atom_ptr"]) - 1 for b in subs]
    rep = pk.temperature_counts(sizes, 2.0)
    osub, osam = pk.build_epoch_index(rep, sizes, seed=5)
    pools = pk.concat(subs)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    ids = offs[osub] + osam
    pool = pk.select(pools, ids)
    atoms = np.diff(pool["atom_ptr"])
    D = CFG["heads"]
    table = dict(rho=np.zeros((D, 119)), rho_has=np.zeros((D, 119), np.uint8), mean=np.zeros(D), std=np.ones(D),
                 fstd=np.ones(D), has=np.ones(D, np.uint8))
    t0 = fit_table(subs[0], D)
    for key in table:
        table[key][0] = t0[key][0]
    table["fstd"][2] = 0.3
    dev = pk.Device(mcfg, seed=7)
    dev.set_option("rank_local", 1)
    dev.set_reference_table(table)
    out = {"workload": ("cfg3: E+F / energy-only / denoising subsets of periodic crystals (8-200 atoms; "
                        "cells of 4.6-14 A: image pairs below 2 rc, minimum image above)" if periodic else
                        "cfg3: E+F / energy-only / denoising subsets (8-200 atoms, non-periodic twin)") +
                       ", T = 2 mix, G = 8, B = 32",
           "epoch_samples": int(len(ids)), "subset_share": [float(np.mean(osub == k)) for k in range(3)],
           "pool_atoms_mean": float(atoms.mean())}
    for mode in ("balanced", "naive"):
        sched = pk.plan(atoms, G, B, 100, seed=3, mode=mode)
        out[mode] = slice_summary(time_rank_slices(pk, dev, pool, sched, G, B, tc, steps))
    dev.close()
    return out


def run_reference(args, dist):
    """--impl reference: the reference's own CPU step (oracle/_ref, the unmodified
    reference compiled from its sources) on this box's host cores, over the same
    cfg2 device-batches (full 256 molecules), workload built by the reference's
    own generator and planner - nothing of the product is imported. Value: all
    host threads, median over the timed steps; one_core: taskset to one core,
    threads = 1 (the sequential run_loop, S/trainer.cpp:262)."""
    lib, batches, table, cfg = reference_workload()
    threads = len(os.sched_getaffinity(0))
    time_reference_steps(lib, batches, table, cfg, threads, max(args.warmup, 1))
    steps = max(args.steps, 5)
    secs, atoms = time_reference_steps(lib, batches, table, cfg, threads, steps)
    rates = [a / s for a, s in zip(atoms, secs)]
    value = float(np.median(rates))
    s1, a1 = time_reference_steps(lib, batches, table, cfg, 1, 5, pin_core=sorted(os.sched_getaffinity(0))[0])
    one = float(np.median([a / s for a, s in zip(a1, s1)]))
    kind = "reference" if lib.kind == "ref" else "port"
    desc = (f"full cfg2 steps (256 molecules, {int(np.mean(atoms))} atoms mean), median of {steps} steps, "
            f"{'oracle/_ref lref_train_step (the unmodified reference)' if kind == 'reference' else 'oracle port'} "
            f"with {threads} threads")
    ms = float(np.median(secs)) * 1e3
    n_gpus = int(os.environ.get("WORLD_SIZE", "1"))
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "atoms/s", "n_gpus": n_gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2: mixed organic molecules 5-60 atoms, batch 256 per GPU, non-periodic",
                       "model": "LaMM MPNN hidden128 layers3 rbf16 cutoff5 heads10", "parallelism": "host threads",
                       "global_batch": BATCH_PER_GPU},
            "cpu_baseline": {"value": value, "unit": "atoms/s", "cores": threads if kind == "reference" else 1,
                             "kind": kind, "sample": desc},
            "one_core": {"value": one, "unit": "atoms/s", "cores": 1, "median_of": 5,
                         "sample": "taskset to one core, threads = 1 (the reference's sequential run_loop)"},
            "host": cpu_info(),
            "e2e": {"value": value, "unit": "atoms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-imbalance", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the larger-than-L2 roofline section")
    ap.add_argument("--only-large", action="store_true", help="run only the larger-than-L2 roofline section")
    ap.add_argument("--only-cost", action="store_true", help="run only the cost-model balancing section")
    ap.add_argument("--only-sweep", action="store_true", help="run only the batch-size sweep")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.impl == "reference":
        # rank 0 alone times the reference on the host cores; no process group,
        # nothing of the product package is imported on this arm
        if int(os.environ.get("RANK", "0")) != 0:
            return
        out = run_reference(args, None)
        assert "paper_2505_22208_b200" not in sys.modules, "the reference arm imported the product"
        out["product_imported"] = False
        print(json.dumps(out), flush=True)
        return
    if args.only_sweep:
        import paper_2505_22208_b200 as pk
        print(json.dumps(batch_sweep(pk, pk.ModelConfig(**CFG), pk.TrainConfig(seed=11))), flush=True)
        return
    if args.only_cost:
        import paper_2505_22208_b200 as pk
        print(json.dumps(cost_balancing(pk, pk.ModelConfig(**CFG), pk.TrainConfig(seed=11))), flush=True)
        return
    if args.only_large:
        import paper_2505_22208_b200 as pk
        print(json.dumps(roofline_large(pk, pk.ModelConfig(**CFG), pk.TrainConfig(seed=11))), flush=True)
        return
    from paper_2505_22208_b200.dist import Dist
    dist = Dist("gloo")
    try:
        out = run_ours(args, dist)
        if out is not None and dist.rank == 0:
            print(json.dumps(out), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
