"""Host-side mirror of the reference's C++ API for the train-step path.

Thin numpy wrappers over the C ABI (include/lamm_b200.h); every computation
runs in liblamm_b200.so — host C++ for the scheduler/generators, sm_100a CUDA
kernels for the model, loss and optimizer. Names and argument meaning follow
the reference (H = /root/reference/proj/core/include/lamm):

* ``init_params``                       H/model.hpp:72
* ``Device.build_neighbor_list``        H/core.hpp:83
* ``Device.forward`` / ``backward``     H/model.hpp:123-129
* ``Device.masked_loss_grad``           H/loss.hpp:81-84
* ``Device.train_step``                 S/trainer.cpp:258-327 (no public reference entry)
* ``greedy_assign`` / ``plan`` / ``schedule_metrics``   H/scheduler.hpp:66-91
* ``make_trace``                        H/trace.hpp:39
* ``temperature_counts`` / ``build_epoch_index`` / ``synth_generate``  H/dataset.hpp:56-138

Batches are dicts of numpy arrays (packed CSR over atoms)::

    atom_ptr int64[B+1], pos f64[N,3], Z int32[N], dataset_index int32[B],
    energy_mask u8[B], force_mask u8[B], energy f64[B], forces f64[N,3], denoise u8[B]
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import (BatchViewC, CostModelC, NormalizerC, SimCostC, SimTotalsC, EvalResultC, InputError, LossBreakdownC, LossConfigC, ModelConfigC, NonFiniteError,  # noqa: F401
                   RefTableC, StepResultC, TrainConfigC, check, lib)


def _p(a):
    return None if a is None else C.c_void_p(a.__array_interface__["data"][0])


def _c(a, dt):
    if isinstance(a, np.ndarray) and a.dtype == dt and a.flags.c_contiguous:
        return a  # the per-step fast path: no copy, no conversion
    return np.ascontiguousarray(a, dtype=dt)


@dataclass(frozen=True)
class ModelConfig:
    """lamm::model::ModelConfig (H/model.hpp:34-40)."""
    hidden: int = 64
    layers: int = 2
    rbf: int = 16
    cutoff: float = 5.0
    heads: int = 1

    def c(self) -> ModelConfigC:
        return ModelConfigC(self.hidden, self.layers, self.rbf, self.heads, self.cutoff)

    def astuple(self):
        return (self.hidden, self.layers, self.rbf, self.cutoff, self.heads)


@dataclass
class LossConfig:
    """lamm::loss::LossConfig (H/loss.hpp:26-29)."""
    lambda_energy: float = 1.0
    lambda_force: float = 1.0


@dataclass
class TrainConfig:
    """Step-body fields of lamm::trainer::TrainConfig (H/trainer.hpp:33-50)."""
    learning_rate: float = 1e-3
    clip_norm: float = 10.0
    rms_decay: float = 0.99
    rms_epsilon: float = 1e-8
    noise_sigma: float = 0.3
    noise_scheme: str = "centered"
    seed: int = 0
    lambda_energy: float = 1.0
    lambda_force: float = 1.0

    def c(self) -> TrainConfigC:
        return TrainConfigC(self.learning_rate, self.clip_norm, self.rms_decay, self.rms_epsilon, self.noise_sigma,
                            1 if self.noise_scheme == "centered" else 0, self.seed, self.lambda_energy,
                            self.lambda_force)


def param_count(cfg: ModelConfig) -> int:
    mc = cfg.c()
    return int(lib().lamm_param_count(C.byref(mc)))


def init_params(cfg: ModelConfig, seed: int) -> np.ndarray:
    """lamm::model::init_params — bit-exact with the reference."""
    out = np.empty(param_count(cfg), np.float64)
    mc = cfg.c()
    check(lib().lamm_init_params(C.byref(mc), C.c_uint64(seed), _p(out)))
    return out


def _batch_view(b: dict):
    ap = _c(b["atom_ptr"], np.int64)
    B = len(ap) - 1

    def opt(key, dt, shape):  # optional per-sample / per-atom arrays (zeros when absent)
        v = b.get(key)
        return _c(v, dt) if v is not None else np.zeros(shape, dt)

    keep = {
        "atom_ptr": ap, "pos": _c(b["pos"], np.float64), "Z": _c(b["Z"], np.int32),
        "dataset_index": opt("dataset_index", np.int32, B), "energy_mask": opt("energy_mask", np.uint8, B),
        "force_mask": opt("force_mask", np.uint8, B), "energy": opt("energy", np.float64, B),
        "forces": opt("forces", np.float64, (len(b["Z"]), 3)), "denoise": opt("denoise", np.uint8, B),
    }
    if b.get("cell") is not None:  # periodic cells [B, 3, 3] (all-zero: non-periodic sample)
        keep["cell"] = _c(np.asarray(b["cell"]).reshape(B, 9), np.float64)
        if b.get("pbc") is not None:  # per-axis periodicity [B, 3] (absent: all periodic)
            keep["pbc"] = _c(np.asarray(b["pbc"]).reshape(B, 3), np.uint8)

    def addr(k):  # c_void_p structure fields take the integer address directly
        return keep[k].__array_interface__["data"][0]

    v = BatchViewC(B, int(ap[-1]), addr("atom_ptr"), addr("pos"), addr("Z"), addr("dataset_index"),
                   addr("energy_mask"), addr("force_mask"), addr("energy"), addr("forces"), addr("denoise"),
                   addr("cell") if "cell" in keep else None, addr("pbc") if "pbc" in keep else None)
    return v, keep


def _table_view(t: dict):
    keep = {k: _c(t[k], dt) for k, dt in (("rho", np.float64), ("rho_has", np.uint8), ("mean", np.float64),
                                          ("std", np.float64), ("fstd", np.float64), ("has", np.uint8))}
    v = RefTableC(len(keep["mean"]), _p(keep["rho"]), _p(keep["rho_has"]), _p(keep["mean"]), _p(keep["std"]),
                  _p(keep["fstd"]), _p(keep["has"]))
    return v, keep


def cell_inverse(cell) -> np.ndarray:
    """The 3x3 cofactor inverse the minimum-image test uses (lamm_cell_inverse)."""
    out = np.empty(9)
    check(lib().lamm_cell_inverse(_p(_c(np.asarray(cell).reshape(9), np.float64)), _p(out)))
    return out


def empty_table(n: int) -> dict:
    """A ReferenceTable with no reference energies, zero mean and unit scales."""
    return dict(rho=np.zeros((n, 119)), rho_has=np.zeros((n, 119), np.uint8), mean=np.zeros(n), std=np.ones(n),
                fstd=np.ones(n), has=np.ones(n, np.uint8))


@dataclass
class StepResult:
    loss: float
    grad_norm: float
    local: dict
    n_atoms: int
    n_edges: int
    status: int
    h2d_bytes: int = 0
    d2h_bytes: int = 0


def _breakdown(b: LossBreakdownC) -> dict:
    return dict(total=b.total, energy_term=b.energy_term, force_term=b.force_term, energy_labeled=b.energy_labeled,
                force_labeled=b.force_labeled, energy_empty=bool(b.energy_empty), force_empty=bool(b.force_empty))


class Device:
    """One lamm_ctx: a model replica on one GPU (one CUDA stream)."""

    def __init__(self, cfg: ModelConfig, device: int = 0, params: np.ndarray | None = None, seed: int = 0):
        self.cfg = cfg
        self._h = C.c_void_p()
        mc = cfg.c()
        check(lib().lamm_ctx_create(device, C.byref(mc), C.byref(self._h)))
        self.n_params = param_count(cfg)
        self.set_params(init_params(cfg, seed) if params is None else params)
        self._batch = None
        self._keep = None

    def close(self):
        if self._h:
            lib().lamm_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, name: str, value: int):
        check(lib().lamm_ctx_set_option(self._h, name.encode(), C.c_int64(int(value))))

    # ---------------------------------------------------------- parameters
    def set_params(self, flat):
        flat = _c(flat, np.float64)
        check(lib().lamm_params_set(self._h, _p(flat), C.c_size_t(len(flat))))

    def params(self) -> np.ndarray:
        out = np.empty(self.n_params)
        check(lib().lamm_params_get(self._h, _p(out), C.c_size_t(self.n_params)))
        return out

    def set_rms_state(self, flat):
        flat = _c(flat, np.float64)
        check(lib().lamm_rms_state_set(self._h, _p(flat), C.c_size_t(len(flat))))

    def rms_state(self) -> np.ndarray:
        out = np.empty(self.n_params)
        check(lib().lamm_rms_state_get(self._h, _p(out), C.c_size_t(self.n_params)))
        return out

    # --------------------------------------------------------------- batch
    def set_reference_table(self, table: dict | None):
        if table is None:
            check(lib().lamm_ref_table_set(self._h, None))
            return
        v, self._tkeep = _table_view(table)
        check(lib().lamm_ref_table_set(self._h, C.byref(v)))

    def set_batch(self, batch: dict):
        v, keep = _batch_view(batch)
        check(lib().lamm_batch_set(self._h, C.byref(v)))
        self._batch, self._keep = batch, keep
        self.B = len(keep["atom_ptr"]) - 1
        self.N = int(keep["atom_ptr"][-1])

    def evaluate(self, batch: dict) -> dict:
        """trainer::evaluate (S/trainer.cpp:528-553): MAEs in meV of the current
        parameters on `batch` (raw labels; replaces the current batch)."""
        v, keep = _batch_view(batch)
        r = EvalResultC()
        check(lib().lamm_evaluate(self._h, C.byref(v), C.byref(r)))
        self._batch, self._keep = batch, keep
        self.B = len(keep["atom_ptr"]) - 1
        self.N = int(keep["atom_ptr"][-1])
        return dict(energy_mae=r.energy_mae, force_mae=r.force_mae, energy_count=r.energy_count,
                    force_count=r.force_count)

    def labels(self):
        e, f = np.empty(self.B), np.empty((self.N, 3))
        check(lib().lamm_labels_get(self._h, _p(e), _p(f)))
        return e, f

    def build_neighbor_list(self, fp64: bool = True):
        """Per-sample pair lists: (sample_pair_ptr, i, j, dist, unit); i/j local."""
        P = C.c_int64()
        check(lib().lamm_neighbor_list(self._h, C.byref(P)))
        P = P.value
        ptr = np.empty(self.B + 1, np.int64)
        oi, oj = np.empty(P, np.int32), np.empty(P, np.int32)
        dist = np.empty(P) if fp64 else None
        unit = np.empty((P, 3)) if fp64 else None
        check(lib().lamm_neighbor_list_copy(self._h, _p(ptr), _p(oi), _p(oj), _p(dist), _p(unit)))
        return ptr, oi, oj, dist, unit

    # ---------------------------------------------------------------- model
    def forward(self):
        """Energies [B, D] and forces (reference Prediction layout, flat)."""
        e = np.empty((self.B, self.cfg.heads))
        f = np.empty(3 * self.cfg.heads * self.N)
        check(lib().lamm_forward(self._h, _p(e), _p(f)))
        return e, f

    def forward_cache(self, which: str, layer: int) -> np.ndarray:
        out = np.empty((self.N, self.cfg.hidden))
        check(lib().lamm_forward_cache_get(self._h, 0 if which == "h" else 1, layer, _p(out)))
        return out

    def masked_loss_grad(self, lcfg: LossConfig | None = None):
        lcfg = lcfg or LossConfig()
        bd = LossBreakdownC()
        ge = np.empty((self.B, self.cfg.heads))
        gf = np.empty(3 * self.cfg.heads * self.N)
        lc = LossConfigC(lcfg.lambda_energy, lcfg.lambda_force)
        check(lib().lamm_loss_grad(self._h, C.byref(lc), C.byref(bd), _p(ge), _p(gf)))
        return _breakdown(bd), ge, gf

    def backward(self, up_energy=None, up_forces=None, grads=None) -> np.ndarray:
        """Accumulates the batch parameter gradient into ``grads`` (fp64)."""
        g = np.zeros(self.n_params) if grads is None else grads
        ue = None if up_energy is None else _c(up_energy, np.float64)
        uf = None if up_forces is None else _c(up_forces, np.float64)
        if (ue is None) != (uf is None):
            ue = np.zeros((self.B, self.cfg.heads)) if ue is None else ue
            uf = np.zeros(3 * self.cfg.heads * self.N) if uf is None else uf
        check(lib().lamm_backward(self._h, _p(ue), _p(uf), _p(g)))
        return g

    def grads(self) -> np.ndarray:
        out = np.empty(self.n_params)
        check(lib().lamm_grads_get(self._h, _p(out), C.c_size_t(self.n_params)))
        return out

    # ----------------------------------------------------------- training
    def last_step_compute_ms(self) -> float:
        """Upload -> allreduce device time of the last synced step (communicator only)."""
        ms = C.c_double()
        check(lib().lamm_last_step_compute_ms(self._h, C.byref(ms)))
        return ms.value

    def comm_init(self, nranks: int, rank: int, unique_id: bytes):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib().lamm_comm_init(self._h, nranks, rank, buf))

    def train_step(self, batch: dict, tcfg: TrainConfig, step: int, workers: int = 1, rank: int = 0) -> StepResult:
        v, keep = _batch_view(batch)
        res = StepResultC()
        tc = tcfg.c()
        st = lib().lamm_train_step(self._h, C.byref(v), C.byref(tc), C.c_int64(step), workers, rank, C.byref(res))
        self._keep = keep
        self.B = len(keep["atom_ptr"]) - 1
        self.N = int(keep["atom_ptr"][-1])
        check(st)
        return StepResult(res.loss, res.grad_norm, _breakdown(res.local), res.n_atoms, res.n_edges, res.status,
                          res.h2d_bytes, res.d2h_bytes)

    def train_step_submit(self, batch: dict, tcfg: TrainConfig, step: int, workers: int = 1, rank: int = 0) -> int:
        """Pipelined train step (lamm_train_step_submit): packs and enqueues the
        step without waiting; returns the ticket for train_step_wait. At most two
        in flight, waited for in order."""
        v, keep = _batch_view(batch)
        tc = tcfg.c()
        t = C.c_int64()
        check(lib().lamm_train_step_submit(self._h, C.byref(v), C.byref(tc), C.c_int64(step), workers, rank,
                                           C.byref(t)))
        return t.value

    def train_step_wait(self, ticket: int) -> StepResult:
        """Waits for the oldest submitted step and returns its result."""
        res = StepResultC()
        check(lib().lamm_train_step_wait(self._h, C.c_int64(ticket), C.byref(res)))
        return StepResult(res.loss, res.grad_norm, _breakdown(res.local), res.n_atoms, res.n_edges, res.status,
                          res.h2d_bytes, res.d2h_bytes)

    def train_steps_pipelined(self, batches, tcfg: TrainConfig, steps, workers: int = 1, rank: int = 0):
        """Runs the steps (batch, step index) in order, the host packing step k+1
        while the device runs step k; returns the results in order."""
        out, pending = [], None
        for b, st in zip(batches, steps):
            t = self.train_step_submit(b, tcfg, st, workers, rank)
            if pending is not None:
                out.append(self.train_step_wait(pending))
            pending = t
        if pending is not None:
            out.append(self.train_step_wait(pending))
        return out

    def train_step_workers(self, batches, tcfg: TrainConfig, step: int) -> StepResult:
        """One optimizer step over G SIMULATED workers on this device
        (S/trainer.cpp:262-319): ``batches[g]`` is worker g's device-batch."""
        G = len(batches)
        views = (BatchViewC * G)()
        keeps = []
        for g, b in enumerate(batches):
            v, keep = _batch_view(b)
            views[g] = v
            keeps.append(keep)
        res = StepResultC()
        tc = tcfg.c()
        st = lib().lamm_train_step_workers(self._h, views, G, C.byref(tc), C.c_int64(step), C.byref(res))
        self._keep = keeps[-1]
        self.B = len(keeps[-1]["atom_ptr"]) - 1
        self.N = int(keeps[-1]["atom_ptr"][-1])
        check(st)
        return StepResult(res.loss, res.grad_norm, _breakdown(res.local), res.n_atoms, res.n_edges, res.status,
                          res.h2d_bytes, res.d2h_bytes)

    def stage(self, batch: dict, tcfg: TrainConfig, step: int, slot: int, workers: int = 1, rank: int = 0) -> int:
        """Packs a device-batch into HBM slot ``slot`` (inputs resident for timing);
        returns the staged blob size in bytes."""
        v, keep = _batch_view(batch)
        tc = tcfg.c()
        check(lib().lamm_stage(self._h, C.byref(v), C.byref(tc), C.c_int64(step), workers, rank, slot))
        return int(keep["atom_ptr"][-1])

    def train_step_staged(self, slot: int, sync: bool = True, next_slot: int | None = None) -> StepResult | None:
        """One step of a staged slot. next_slot: also build that slot's batch preparation
        (denoise, labels, neighbour list) on a side stream during this step's model
        (lamm_train_step_staged_next); the next call with slot == next_slot uses it."""
        res = StepResultC()
        if next_slot is None:
            check(lib().lamm_train_step_staged(self._h, slot, 1 if sync else 0, C.byref(res) if sync else None))
        else:
            check(lib().lamm_train_step_staged_next(self._h, slot, next_slot, 1 if sync else 0,
                                                    C.byref(res) if sync else None))
        if not sync:
            return None
        return StepResult(res.loss, res.grad_norm, _breakdown(res.local), res.n_atoms, res.n_edges, res.status)

    def anomalies(self) -> int:
        return int(lib().lamm_anomalies(self._h))

    def flush_l2(self, nbytes: int = 256 << 20):
        check(lib().lamm_flush_l2(self._h, C.c_int64(nbytes)))

    def optimizer_step(self, grad_sum, workers: int, tcfg: TrainConfig) -> float:
        g = _c(grad_sum, np.float64)
        gn = C.c_double()
        tc = tcfg.c()
        check(lib().lamm_optimizer_step(self._h, _p(g), workers, C.byref(tc), C.byref(gn)))
        return gn.value

    # --------------------------------------------------------------- timing
    def sync(self):
        check(lib().lamm_sync(self._h))

    def event_record(self, slot: int):
        check(lib().lamm_event_record(self._h, slot))

    def event_elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        check(lib().lamm_event_elapsed_ms(self._h, a, b, C.byref(ms)))
        return ms.value

    def kernel_times(self) -> dict:
        n = C.c_int()
        check(lib().lamm_kernel_times(self._h, 0, None, None, None, C.byref(n)))
        k = n.value
        names = (C.c_char_p * max(k, 1))()
        ms = np.zeros(max(k, 1))
        cnt = np.zeros(max(k, 1), np.int64)
        check(lib().lamm_kernel_times(self._h, k, names, _p(ms), _p(cnt), C.byref(n)))
        return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(k)}

    def step_times(self):
        """(total device ms, steps) of the synced train steps since the last reset."""
        ms, n = C.c_double(), C.c_int64()
        check(lib().lamm_step_times(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def kernel_times_reset(self):
        check(lib().lamm_kernel_times_reset(self._h))

    def info(self, name: str) -> int:
        """Launch geometry (lamm_ctx_get_info): grid_edge, parts_per_cta, chunk_edges, ..."""
        v = C.c_int64()
        check(lib().lamm_ctx_get_info(self._h, name.encode(), C.byref(v)))
        return v.value

    def last_step_launches(self) -> int:
        return int(lib().lamm_last_step_launches(self._h))


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().lamm_comm_unique_id(buf))
    return buf.raw


# ------------------------------------------------------------ host: schedule
MODES = {"balanced": 0, "greedy_only": 1, "naive": 2}


def greedy_assign(atoms, workers: int, batch_per_worker: int) -> np.ndarray:
    a = _c(atoms, np.int64)
    out = np.empty(len(a), np.int32)
    check(lib().lamm_greedy_assign(_p(a), C.c_int64(len(a)), workers, batch_per_worker, _p(out)))
    return out


def plan(atoms, workers: int, batch_per_worker: int, num_splits: int = 100, seed: int = 0,
         mode: str = "balanced") -> dict:
    """lamm::scheduler::plan + schedule_metrics, as flat ScheduledSample arrays."""
    a = _c(atoms, np.int64)
    n = len(a)
    cap = max(n, 1)
    out = dict(sample=np.empty(cap, np.int64), worker=np.empty(cap, np.int32), atoms=np.empty(cap, np.int64),
               split=np.empty(cap, np.int64), chunk_rank=np.empty(cap, np.int64),
               worker_atoms=np.empty(cap, np.int64))
    nb, dr = C.c_int64(), C.c_int64()
    check(lib().lamm_plan(_p(a), C.c_int64(n), workers, batch_per_worker, num_splits, C.c_uint64(seed), MODES[mode],
                          _p(out["sample"]), _p(out["worker"]), _p(out["atoms"]), _p(out["split"]),
                          _p(out["chunk_rank"]), _p(out["worker_atoms"]), C.byref(nb), C.byref(dr)))
    nb, dr = nb.value, dr.value
    tot = nb * workers * batch_per_worker
    for k in ("sample", "worker", "atoms", "split", "chunk_rank"):
        out[k] = out[k][:tot]
    out["worker_atoms"] = out["worker_atoms"][:nb * workers]
    mx, mean, mono, grow = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
    check(lib().lamm_schedule_metrics(C.c_int64(nb), workers, batch_per_worker, _p(out["worker"]), _p(out["atoms"]),
                                      _p(out["split"]), _p(out["chunk_rank"]), C.byref(mx), C.byref(mean),
                                      C.byref(mono), C.byref(grow)))
    out.update(n_batches=nb, dropped=dr, max_imbalance=mx.value, mean_imbalance=mean.value,
               monotonicity_violations=mono.value, growth_events=grow.value)
    return out


@dataclass
class CostModel:
    """Predicted per-sample step cost (lamm_cost_model): (per_sample + per_atom *
    atoms) + per_edge * edges. CostModel(0, 1, 0) is the reference's atom count."""
    per_sample: float = 0.0
    per_atom: float = 1.0
    per_edge: float = 0.0

    def c(self):
        return CostModelC(self.per_sample, self.per_atom, self.per_edge)


def sample_cost(atoms, edges, model: CostModel) -> np.ndarray:
    a = _c(atoms, np.int64)
    e = None if edges is None else _c(edges, np.int64)
    out = np.empty(len(a), np.float64)
    cm = model.c()
    check(lib().lamm_sample_cost(_p(a), _p(e) if e is not None else None, C.c_int64(len(a)), C.byref(cm), _p(out)))
    return out


def plan_cost(atoms, edges, model: CostModel, workers: int, batch_per_worker: int, num_splits: int = 100,
              seed: int = 0, mode: str = "balanced") -> dict:
    """lamm_plan_cost: the reference's plan with the predicted cost as the balancing
    key (north_star "predicted atom/edge cost"); adds worker_cost [n_batches][G]."""
    a = _c(atoms, np.int64)
    e = None if edges is None else _c(edges, np.int64)
    n = len(a)
    cap = max(n, 1)
    out = dict(sample=np.empty(cap, np.int64), worker=np.empty(cap, np.int32), atoms=np.empty(cap, np.int64),
               split=np.empty(cap, np.int64), chunk_rank=np.empty(cap, np.int64),
               worker_atoms=np.empty(cap, np.int64), worker_cost=np.empty(cap, np.float64))
    nb, dr = C.c_int64(), C.c_int64()
    cm = model.c()
    check(lib().lamm_plan_cost(_p(a), _p(e) if e is not None else None, C.c_int64(n), C.byref(cm), workers,
                               batch_per_worker, num_splits, C.c_uint64(seed), MODES[mode], _p(out["sample"]),
                               _p(out["worker"]), _p(out["atoms"]), _p(out["split"]), _p(out["chunk_rank"]),
                               _p(out["worker_atoms"]), _p(out["worker_cost"]), C.byref(nb), C.byref(dr)))
    nb, dr = nb.value, dr.value
    tot = nb * workers * batch_per_worker
    for k in ("sample", "worker", "atoms", "split", "chunk_rank"):
        out[k] = out[k][:tot]
    out["worker_atoms"] = out["worker_atoms"][:nb * workers]
    out["worker_cost"] = out["worker_cost"][:nb * workers]
    wc = out["worker_cost"].reshape(nb, workers) if nb else np.ones((1, workers))
    out.update(n_batches=nb, dropped=dr,
               cost_imbalance_mean=float(np.mean(wc.max(1) / wc.mean(1))) if nb else 1.0)
    return out


def fit_cost_model(atoms, edges, times, samples=None) -> tuple:
    """Non-negative least-squares step-time model t = t0 + per_atom * atoms +
    per_edge * edges (+ per_sample * samples when given) over measured per-rank steps; returns
    (CostModel, t0, r2). t0 (the per-step fixed cost) is the same on every rank and
    does not enter the balancing."""
    cols = [np.ones(len(times)), np.asarray(atoms, float), np.asarray(edges, float)]
    if samples is not None:
        cols.append(np.asarray(samples, float))
    A = np.stack(cols, 1)
    y = np.asarray(times, float)
    # non-negative least squares (a cost cannot fall with atoms or edges; atoms and
    # edges are strongly correlated, so an unconstrained fit can trade them off)
    from scipy.optimize import nnls
    scale = np.maximum(np.abs(A).max(0), 1e-300)
    coef, _ = nnls(A / scale, y)
    coef = coef / scale
    pred = A @ coef
    r2 = 1.0 - float(np.sum((y - pred) ** 2) / max(np.sum((y - y.mean()) ** 2), 1e-300))
    cm = CostModel(per_sample=float(coef[3]) if samples is not None else 0.0, per_atom=float(coef[1]),
                   per_edge=float(coef[2]))
    return cm, float(coef[0]), r2


# ------------------------------------------------------- data layer (host C++)
def filter_max_atoms(atom_ptr, limit: int) -> np.ndarray:
    """dataset::filter_max_atoms (S/dataset.cpp:85-96): kept sample indices."""
    ap = _c(atom_ptr, np.int64)
    out = np.empty(max(len(ap) - 1, 1), np.int64)
    n = C.c_int64()
    check(lib().lamm_filter_max_atoms(_p(ap), C.c_int64(len(ap) - 1), C.c_int64(limit), _p(out), C.byref(n)))
    return out[:n.value]


def split_train_val(n: int, val_fraction: float, seed: int):
    """dataset::split_train_val (S/dataset.cpp:98-111): (train ids, val ids)."""
    tr, va = np.empty(max(n, 1), np.int64), np.empty(max(n, 1), np.int64)
    nt, nv = C.c_int64(), C.c_int64()
    check(lib().lamm_split_train_val(C.c_int64(n), C.c_double(val_fraction), C.c_uint64(seed), _p(tr),
                                     C.byref(nt), _p(va), C.byref(nv)))
    return tr[:nt.value], va[:nv.value]


def apply_noise(positions, sigma: float, scheme: int, seed: int):
    """denoise::apply_noise (S/denoise.cpp:7-40): (noisy positions, pseudo-forces)."""
    pos = _c(positions, np.float64).reshape(-1, 3)
    noisy, pf = np.empty_like(pos), np.empty_like(pos)
    check(lib().lamm_apply_noise(_p(pos), C.c_int64(len(pos)), C.c_double(sigma), scheme, C.c_uint64(seed),
                                 _p(noisy), _p(pf)))
    return noisy, pf


def pseudo_force_std(batch: dict, sigma: float, scheme: int, seed: int, ids=None) -> float:
    """estimate_pseudo_force_std (S/trainer.cpp:82-100) over ids (default: all samples)."""
    ap = _c(batch["atom_ptr"], np.int64)
    pos = _c(batch["pos"], np.float64)
    idv = None if ids is None else _c(ids, np.int64)
    n = len(ap) - 1 if ids is None else len(idv)
    out = C.c_double()
    check(lib().lamm_pseudo_force_std(_p(ap), _p(pos), _p(idv) if idv is not None else None, C.c_int64(n),
                                      C.c_double(sigma), scheme, C.c_uint64(seed), C.byref(out)))
    return out.value


def fit_normalizer(batch: dict, pseudo_force_std: float = 0.0) -> dict:
    """loss::fit_normalizer (S/loss.cpp:64-111): rho [119] (by Z), rho_has, mean, std,
    fstd, has (one row of a reference table)."""
    v, keep = _batch_view(batch)
    out = NormalizerC()
    check(lib().lamm_fit_normalizer(C.byref(v), C.c_double(pseudo_force_std), C.byref(out)))
    return dict(rho=np.array(out.rho[:]), rho_has=np.array(out.rho_has[:], np.uint8), mean=out.energy_mean,
                std=out.energy_std, fstd=out.force_std, has=int(out.has_energy_stats))


def init_heads(cfg: ModelConfig, heads: int, seed: int):
    """model::reset_heads' fresh heads (S/model.cpp:167-202): (energy_head [H, heads],
    force_head [2H+K, heads])."""
    H, K = cfg.hidden, cfg.rbf
    e, f = np.empty(H * heads), np.empty((2 * H + K) * heads)
    mc = cfg.c()
    check(lib().lamm_init_heads(C.byref(mc), heads, C.c_uint64(seed), _p(e), _p(f)))
    return e.reshape(H, heads), f.reshape(2 * H + K, heads)


def simulate(schedule: dict, alpha_s=0.005, beta_s_per_atom=1e-5, gamma_s=0.010, delta_s=0.050,
             worker_cost=None) -> dict:
    """simulator::simulate (S/simulator.cpp:19-59) of a plan() / plan_cost() schedule:
    per-step time (slowest worker + gamma), idle, realloc events, max worker atoms,
    per-worker idle and totals. worker_cost [n_batches, G] (seconds, optional): the
    cost model's own per-worker prediction in place of alpha + beta * atoms."""
    nb = int(schedule["n_batches"])
    G = len(schedule["worker_atoms"]) // max(nb, 1) if nb else 1
    wa = _c(schedule["worker_atoms"], np.int64)
    per = len(schedule["sample"]) // max(nb, 1) if nb else 0
    wc = None if worker_cost is None else _c(worker_cost, np.float64)
    out = dict(step_time=np.empty(max(nb, 1)), step_idle=np.empty(max(nb, 1)),
               step_realloc=np.empty(max(nb, 1), np.int32), step_max_atoms=np.empty(max(nb, 1), np.int64),
               worker_idle=np.empty(G))
    cost, tot = SimCostC(alpha_s, beta_s_per_atom, gamma_s, delta_s), SimTotalsC()
    check(lib().lamm_simulate(_p(wa), _p(wc) if wc is not None else None, C.c_int64(nb), G, C.c_int64(per),
                              C.byref(cost), _p(out["step_time"]), _p(out["step_idle"]), _p(out["step_realloc"]),
                              _p(out["step_max_atoms"]), _p(out["worker_idle"]), C.byref(tot)))
    for k in ("step_time", "step_idle", "step_realloc", "step_max_atoms"):
        out[k] = out[k][:nb]
    out.update(total_s=tot.total_s, throughput_samples_per_s=tot.throughput_samples_per_s,
               realloc_events=tot.realloc_events, samples=tot.samples)
    return out


TRACE_KINDS = {"constant": 0, "uniform": 1, "lognormal": 2, "bimodal": 3}


def make_trace(kind="lognormal", count=1000, min_atoms=1, max_atoms=300, constant_atoms=15.0, mode=15.0, sigma=0.45,
               mode_a=15.0, sigma_a=0.30, mode_b=160.0, sigma_b=0.30, weight_a=0.5, seed=0) -> np.ndarray:
    out = np.empty(count, np.int64)
    D = C.c_double
    check(lib().lamm_make_trace(TRACE_KINDS[kind], C.c_int64(count), C.c_int64(min_atoms), C.c_int64(max_atoms),
                                D(constant_atoms), D(mode), D(sigma), D(mode_a), D(sigma_a), D(mode_b), D(sigma_b),
                                D(weight_a), C.c_uint64(seed), _p(out)))
    return out


def temperature_counts(sizes, temperature: float) -> np.ndarray:
    s = _c(sizes, np.float64)
    out = np.empty(len(s))
    check(lib().lamm_temperature_counts(_p(s), len(s), C.c_double(temperature), _p(out)))
    return out


def build_epoch_index(repeats, sizes, seed: int):
    r, s = _c(repeats, np.float64), _c(sizes, np.int64)
    cap = int(sum(int(np.rint(x)) for x in r)) + 8
    osub, osam = np.empty(cap, np.int32), np.empty(cap, np.int64)
    cnt = C.c_int64()
    check(lib().lamm_build_epoch_index(_p(r), _p(s), len(s), C.c_uint64(seed), C.c_int64(cap), _p(osub), _p(osam),
                                       C.byref(cnt)))
    return osub[:cnt.value], osam[:cnt.value]


TASKS = {"energy_and_forces": 0, "energy_only": 1, "denoising": 2}


def synth_generate(count: int, seed: int, *, task="energy_and_forces", mode=15.0, sigma=0.45, min_atoms=2,
                   max_atoms=300, elements=(6,), relax_steps=6, relax_step=0.02, energy_scale=1.0, offsets=None,
                   threads: int = 8, dataset_index: int = 0) -> dict:
    """lamm::dataset::synth_generate (Morse clusters) as a packed batch dict."""
    el = _c(list(elements), np.int32)
    offsets = offsets or {}
    oz = _c(list(offsets.keys()) or [0], np.int32)
    ov = _c(list(offsets.values()) or [0.0], np.float64)
    ap = np.empty(count + 1, np.int64)
    D = C.c_double
    check(lib().lamm_synth_counts(C.c_int64(count), D(mode), D(sigma), min_atoms, max_atoms, C.c_uint64(seed),
                                  _p(ap)))
    N = int(ap[-1])
    b = dict(atom_ptr=ap, pos=np.empty((N, 3)), Z=np.empty(N, np.int32), energy_mask=np.empty(count, np.uint8),
             force_mask=np.empty(count, np.uint8), energy=np.empty(count), forces=np.empty((N, 3)))
    check(lib().lamm_synth_fill(TASKS[task], C.c_int64(count), D(mode), D(sigma), min_atoms, max_atoms, _p(el),
                                len(el), relax_steps, D(relax_step), D(energy_scale), _p(oz), _p(ov), len(offsets),
                                C.c_uint64(seed), threads, _p(ap), _p(b["pos"]), _p(b["Z"]), _p(b["energy_mask"]),
                                _p(b["force_mask"]), _p(b["energy"]), _p(b["forces"])))
    b["dataset_index"] = np.full(count, dataset_index, np.int32)
    b["denoise"] = np.full(count, 1 if task == "denoising" else 0, np.uint8)
    return b


def mix_seed(a: int, b: int) -> int:
    return int(lib().lamm_mix_seed(a, b))


def rng_normals(seed: int, n: int) -> np.ndarray:
    out = np.empty(n)
    check(lib().lamm_rng_normals(C.c_uint64(seed), C.c_int64(n), _p(out)))
    return out


def select(batch: dict, ids) -> dict:
    """Packs the samples ``ids`` (in order) of a batch dict into a new batch."""
    ap = batch["atom_ptr"]
    ids = np.asarray(ids, np.int64)
    sizes = ap[ids + 1] - ap[ids]
    nap = np.zeros(len(ids) + 1, np.int64)
    np.cumsum(sizes, out=nap[1:])
    rows = np.concatenate([np.arange(ap[i], ap[i + 1]) for i in ids]) if len(ids) else np.zeros(0, np.int64)
    out = dict(atom_ptr=nap)
    for k in ("pos", "Z", "forces"):
        out[k] = np.ascontiguousarray(batch[k][rows])
    for k in ("dataset_index", "energy_mask", "force_mask", "energy", "denoise"):
        out[k] = np.ascontiguousarray(batch[k][ids])
    if batch.get("cell") is not None:
        out["cell"] = np.ascontiguousarray(np.asarray(batch["cell"]).reshape(-1, 3, 3)[ids])
        if batch.get("pbc") is not None:
            out["pbc"] = np.ascontiguousarray(np.asarray(batch["pbc"]).reshape(-1, 3)[ids])
    return out


def concat(batches) -> dict:
    """Concatenates packed batch dicts sample-wise."""
    batches = list(batches)
    out = {}
    for k in ("pos", "Z", "forces", "dataset_index", "energy_mask", "force_mask", "energy", "denoise"):
        out[k] = np.concatenate([b[k] for b in batches])
    sizes = np.concatenate([np.diff(b["atom_ptr"]) for b in batches])
    out["atom_ptr"] = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    if any(b.get("cell") is not None for b in batches):  # non-periodic parts get all-zero cells
        out["cell"] = np.concatenate([np.asarray(b["cell"]).reshape(-1, 3, 3) if b.get("cell") is not None
                                      else np.zeros((len(b["atom_ptr"]) - 1, 3, 3)) for b in batches])
        if any(b.get("pbc") is not None for b in batches):  # parts without flags: all periodic
            out["pbc"] = np.concatenate([np.asarray(b["pbc"], np.uint8).reshape(-1, 3) if b.get("pbc") is not None
                                         else np.ones((len(b["atom_ptr"]) - 1, 3), np.uint8) for b in batches])
    return out
