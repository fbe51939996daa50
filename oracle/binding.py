"""ctypes bindings for the two CPU checkers (test infrastructure only).

Both libraries export the same function set — ``lref_*`` (the reference itself,
``oracle/_ref/liblamm_ref.so``) and ``lor_*`` (the plain-C restatement,
``oracle/_build/liblamm_oracle.so``) — so :class:`OracleLib` wraps either one
with one numpy-facing API. Batches are dicts of numpy arrays with the packed
layout documented in ``include/lamm_b200.h``::

    atom_ptr int64[B+1], pos f64[N,3], Z int32[N], dataset_index int32[B],
    energy_mask u8[B], force_mask u8[B], energy f64[B], forces f64[N,3],
    denoise u8[B]

Model configs are ``(H, L, K, cutoff, D)`` tuples; reference tables are dicts
with ``rho``/``rho_has`` ([ntab,119]), ``mean``, ``std``, ``fstd``, ``has``.
"""
from __future__ import annotations

import ctypes as C
import contextlib
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(_HERE, "_ref", "liblamm_ref.so")
PORT_PATH = os.path.join(_HERE, "_build", "liblamm_oracle.so")

_i32, _i64, _u64, _f64, _u8 = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_uint8
_P = C.c_void_p


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleError(RuntimeError):
    pass


class OracleLib:
    """Numpy wrapper over ``lref_*`` (kind='ref') or ``lor_*`` (kind='port')."""

    def __init__(self, path: str, kind: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pre = "lref_" if kind == "ref" else "lor_"
        self._f("last_error").restype = C.c_char_p
        self._f("mix_seed").restype = _u64
        self._f("mix_seed").argtypes = [_u64, _u64]
        for nm in ("neighbor_list", "param_count", "build_epoch_index"):
            self._f(nm).restype = _i64
        if kind == "ref":
            self.lib.lref_plan.restype = _P
            self.lib.lref_synth_generate.restype = _P
        else:
            self.lib.lor_plan.restype = _i64

    def _f(self, name):
        # attribute access caches the function object, so restype sticks
        return getattr(self.lib, self.pre + name)

    def _check(self, st):
        if st != 0:
            raise OracleError(f"{self.pre}: status {st}: {self._f('last_error')().decode()}")

    # ----------------------------------------------------- periodic cells
    def cell_inverse(self, cell):
        """lor_cell_inverse (port): the cofactor inverse the minimum image uses."""
        out = np.empty(9, np.float64)
        self._check(self.lib.lor_cell_inverse(_p(_c(np.asarray(cell).reshape(9), np.float64)), _p(out)))
        return out

    @contextlib.contextmanager
    def periodic(self, cells, pbc=None):
        """Port only: batch calls inside use these cells ([B, 3, 3], all-zero = non-periodic)
        and per-axis periodicity pbc ([B, 3], None = all periodic): every image within the
        cutoff (parity-unpinned extension: the reference has no cells)."""
        if self.kind != "port":
            raise NotImplementedError("the reference has no periodic cells")
        cells = _c(np.asarray(cells).reshape(-1, 9), np.float64)
        inv = np.zeros_like(cells)
        for s in range(len(cells)):
            if np.any(cells[s] != 0.0):
                inv[s] = self.cell_inverse(cells[s])
        flags = None if pbc is None else _c(np.asarray(pbc).reshape(-1, 3), np.uint8)
        self.lib.lor_set_cells(_p(cells), _p(inv))
        self.lib.lor_set_pbc(_p(flags) if flags is not None else None)
        try:
            yield
        finally:
            self.lib.lor_set_cells(None, None)
            self.lib.lor_set_pbc(None)

    def _samples_from_handle(self, h):
        cnt, tot = _i64(), _i64()
        self.lib.lref_samples_info(_P(h), C.byref(cnt), C.byref(tot))
        B, N = cnt.value, tot.value
        b = dict(atom_ptr=np.empty(B + 1, np.int64), pos=np.empty((N, 3)), Z=np.empty(N, np.int32),
                 energy_mask=np.empty(B, np.uint8), force_mask=np.empty(B, np.uint8), energy=np.empty(B),
                 forces=np.empty((N, 3)))
        self.lib.lref_samples_copy(_P(h), _p(b["atom_ptr"]), _p(b["pos"]), _p(b["Z"]), _p(b["energy_mask"]),
                                   _p(b["force_mask"]), _p(b["energy"]), _p(b["forces"]))
        return b

    # ------------------------------------------------- on-disk formats (ref)
    def write_demo_catalog(self, directory, count, seed):
        self._check(self.lib.lref_write_demo_catalog(os.fsencode(directory), _i64(count), _u64(seed)))

    def read_catalog(self, directory):
        """lamm::dataset::read_catalog, every subset concatenated: (batch, subset sizes)."""
        self.lib.lref_read_catalog.restype = _P
        ns = C.c_int32()
        sizes = np.zeros(64, np.int64)
        h = self.lib.lref_read_catalog(os.fsencode(directory), C.byref(ns), _p(sizes))
        if not h:
            raise OracleError(self._f("last_error")().decode())
        try:
            b = self._samples_from_handle(h)
            b["dataset_index"] = np.empty(len(b["atom_ptr"]) - 1, np.int32)
            self.lib.lref_samples_heads(_P(h), _p(b["dataset_index"]))
        finally:
            self.lib.lref_samples_free(_P(h))
        return b, sizes[:ns.value]

    def checkpoint_save(self, path, cfg, params):
        H, L, K, rc, D = cfg
        self._check(self.lib.lref_checkpoint_save(os.fsencode(path), H, L, K, _f64(rc), D,
                                                  _p(_c(params, np.float64))))

    def checkpoint_load(self, path, cap=10_000_000):
        c = np.zeros(4, np.int32)
        rc = C.c_double()
        out = np.empty(cap, np.float64)
        self._check(self.lib.lref_checkpoint_load(os.fsencode(path), _p(c), C.byref(rc), _p(out), _i64(cap)))
        H, L, K, D = (int(x) for x in c)
        return (H, L, K, rc.value, D), out[:self.param_count((H, L, K, rc.value, D))]

    # ---------------------------------------------------------------- rng
    def mix_seed(self, a, b):
        return int(self._f("mix_seed")(_u64(a), _u64(b)))

    def rng_normals(self, seed, n):
        o = np.empty(n, np.float64)
        self._f("rng_normals")(_u64(seed), _i64(n), _p(o))
        return o

    def rng_uniforms(self, seed, n):
        o = np.empty(n, np.float64)
        self._f("rng_uniforms")(_u64(seed), _i64(n), _p(o))
        return o

    def rng_u64(self, seed, n):
        o = np.empty(n, np.uint64)
        self._f("rng_u64")(_u64(seed), _i64(n), _p(o))
        return o

    def rng_bounded(self, seed, n, bound):
        o = np.empty(n, np.uint64)
        self._f("rng_bounded")(_u64(seed), _i64(n), _u64(bound), _p(o))
        return o

    def rng_permutation(self, seed, n):
        o = np.empty(n, np.int64)
        self._f("rng_permutation")(_u64(seed), _i64(n), _p(o))
        return o

    # ------------------------------------------------------- data layer (ref)
    def split_train_val(self, n, val_fraction, seed):
        tr, va = np.empty(max(n, 1), np.int64), np.empty(max(n, 1), np.int64)
        nt, nv = _i64(), _i64()
        self._check(self.lib.lref_split_train_val(_i64(n), _f64(val_fraction), _u64(seed), _p(tr), C.byref(nt),
                                                  _p(va), C.byref(nv)))
        return tr[:nt.value], va[:nv.value]

    def fit_normalizer(self, b, pseudo_std=0.0):
        B = len(b["atom_ptr"]) - 1
        rho, has, st = np.zeros(119), np.zeros(119, np.uint8), np.zeros(4)
        self._check(self.lib.lref_fit_normalizer(
            B, _p(_c(b["atom_ptr"], np.int64)), _p(_c(b["pos"], np.float64)), _p(_c(b["Z"], np.int32)),
            _p(_c(b["energy_mask"], np.uint8)), _p(_c(b["force_mask"], np.uint8)), _p(_c(b["energy"], np.float64)),
            _p(_c(b["forces"], np.float64)), _f64(pseudo_std), _p(rho), _p(has), _p(st)))
        return dict(rho=rho, rho_has=has, mean=st[0], std=st[1], fstd=st[2], has=int(st[3]))

    def pseudo_force_std(self, b, sigma, scheme, seed):
        out = C.c_double()
        self._check(self.lib.lref_pseudo_force_std(len(b["atom_ptr"]) - 1, _p(_c(b["atom_ptr"], np.int64)),
                                                   _p(_c(b["pos"], np.float64)), _p(_c(b["Z"], np.int32)),
                                                   _f64(sigma), scheme, _u64(seed), C.byref(out)))
        return out.value

    def simulate(self, worker_atoms, n_batches, G, samples_per_batch, cost4):
        nb = n_batches
        o = dict(step_time=np.empty(max(nb, 1)), step_idle=np.empty(max(nb, 1)),
                 step_realloc=np.empty(max(nb, 1), np.int32), step_max_atoms=np.empty(max(nb, 1), np.int64),
                 worker_idle=np.empty(G), totals=np.empty(4))
        self._check(self.lib.lref_simulate(_p(_c(worker_atoms, np.int64)), _i64(nb), G, _i64(samples_per_batch),
                                           _p(_c(cost4, np.float64)), _p(o["step_time"]), _p(o["step_idle"]),
                                           _p(o["step_realloc"]), _p(o["step_max_atoms"]), _p(o["worker_idle"]),
                                           _p(o["totals"])))
        for k in ("step_time", "step_idle", "step_realloc", "step_max_atoms"):
            o[k] = o[k][:nb]
        return o

    def reset_heads(self, cfg, params, heads, seed):
        H, L, K, rc, D = cfg
        e, f = np.empty(H * heads), np.empty((2 * H + K) * heads)
        self._check(self.lib.lref_reset_heads(H, L, K, _f64(rc), D, _p(_c(params, np.float64)), heads, _u64(seed),
                                              _p(e), _p(f)))
        return e.reshape(H, heads), f.reshape(2 * H + K, heads)

    # ----------------------------------------------------------- geometry
    def neighbor_list(self, pos, Z, cutoff):
        pos = _c(pos, np.float64).reshape(-1, 3)
        Z = _c(Z, np.int32)
        n = len(Z)
        cap = max(1, n * (n - 1))
        while True:  # periodic images can give more than n (n - 1) pairs: grow and retry
            oi, oj = np.empty(cap, np.int32), np.empty(cap, np.int32)
            od, ou = np.empty(cap, np.float64), np.empty((cap, 3), np.float64)
            cnt = self._f("neighbor_list")(_i32(n), _p(pos), _p(Z), _f64(cutoff), _i64(cap), _p(oi), _p(oj),
                                           _p(od), _p(ou))
            if cnt < 0:
                raise OracleError(self._f("last_error")().decode())
            if cnt <= cap:
                return oi[:cnt], oj[:cnt], od[:cnt], ou[:cnt]
            cap = cnt

    # -------------------------------------------------------------- model
    def param_count(self, cfg):
        H, L, K, _, D = cfg
        return int(self._f("param_count")(H, L, K, D))

    def init_params(self, cfg, seed):
        H, L, K, rc, D = cfg
        o = np.empty(self.param_count(cfg), np.float64)
        self._check(self._f("init_params")(H, L, K, _f64(rc), D, _u64(seed), _p(o)))
        return o

    def forward(self, cfg, params, batch):
        H, L, K, rc, D = cfg
        ap = _c(batch["atom_ptr"], np.int64)
        B, N = len(ap) - 1, int(ap[-1])
        pos, Z = _c(batch["pos"], np.float64), _c(batch["Z"], np.int32)
        e = np.empty((B, D), np.float64)
        f = np.empty(3 * D * N, np.float64)
        self._check(self._f("forward")(H, L, K, _f64(rc), D, _p(_c(params, np.float64)), _i32(B), _p(ap), _p(pos),
                                       _p(Z), _p(e), _p(f)))
        return e, f

    def evaluate(self, cfg, params, batch, table):
        """trainer::evaluate (S/trainer.cpp:528-553): physical-unit MAEs (meV)."""
        if self.kind != "ref":
            raise NotImplementedError("evaluate is checked against the compiled reference only")
        H, L, K, rc, D = cfg
        ap = _c(batch["atom_ptr"], np.int64)
        B = len(ap) - 1
        out = np.empty(4, np.float64)
        keep = [_c(batch[k], dt) for k, dt in (("pos", np.float64), ("Z", np.int32), ("dataset_index", np.int32),
                                               ("energy_mask", np.uint8), ("force_mask", np.uint8),
                                               ("energy", np.float64), ("forces", np.float64))]
        self._check(self._f("evaluate")(H, L, K, _f64(rc), D, _p(_c(params, np.float64)), _i32(B), _p(ap),
                                        *[_p(k) for k in keep], *self._table_args(table), _p(out)))
        return dict(energy_mae=out[0], force_mae=out[1], energy_count=int(out[2]), force_count=int(out[3]))

    def forward_cache(self, cfg, params, pos, Z):
        H, L, K, rc, D = cfg
        pos, Z = _c(pos, np.float64), _c(Z, np.int32)
        n = len(Z)
        h = np.empty((L + 1, n, H), np.float64)
        mt = np.empty((max(L, 1), n, H), np.float64)
        self._check(self._f("forward_cache")(H, L, K, _f64(rc), D, _p(_c(params, np.float64)), _i32(n), _p(pos),
                                             _p(Z), _p(h), _p(mt)))
        return h, mt[:L]

    def backward(self, cfg, params, batch, up_e, up_f, grads=None):
        H, L, K, rc, D = cfg
        ap = _c(batch["atom_ptr"], np.int64)
        B = len(ap) - 1
        g = np.zeros(self.param_count(cfg), np.float64) if grads is None else _c(grads, np.float64).copy()
        self._check(self._f("backward")(H, L, K, _f64(rc), D, _p(_c(params, np.float64)), _i32(B), _p(ap),
                                        _p(_c(batch["pos"], np.float64)), _p(_c(batch["Z"], np.int32)),
                                        _p(_c(up_e, np.float64)), _p(_c(up_f, np.float64)), _p(g)))
        return g

    # --------------------------------------------------------------- loss
    @staticmethod
    def _table_args(t):
        ntab = len(t["mean"])
        return (ntab, _p(_c(t["rho"], np.float64)), _p(_c(t["rho_has"], np.uint8)), _p(_c(t["mean"], np.float64)),
                _p(_c(t["std"], np.float64)), _p(_c(t["fstd"], np.float64)), _p(_c(t["has"], np.uint8)))

    def normalize_labels(self, batch, table):
        ap = _c(batch["atom_ptr"], np.int64)
        B, N = len(ap) - 1, int(ap[-1])
        oe, of = np.empty(B, np.float64), np.empty((N, 3), np.float64)
        keep = [_c(batch[k], dt) for k, dt in (("pos", np.float64), ("Z", np.int32), ("dataset_index", np.int32),
                                               ("energy_mask", np.uint8), ("force_mask", np.uint8),
                                               ("energy", np.float64), ("forces", np.float64))]
        self._check(self._f("normalize_labels")(_i32(B), _p(ap), *[_p(k) for k in keep], *self._table_args(table),
                                                _p(oe), _p(of)))
        return oe, of

    def loss_grad(self, batch, D, pred_e, pred_f, lambda_e=1.0, lambda_f=1.0):
        ap = _c(batch["atom_ptr"], np.int64)
        B, N = len(ap) - 1, int(ap[-1])
        bd = np.empty(7, np.float64)
        ge, gf = np.empty((B, D), np.float64), np.empty(3 * D * N, np.float64)
        keep = [_c(batch[k], dt) for k, dt in (("dataset_index", np.int32), ("energy_mask", np.uint8),
                                               ("force_mask", np.uint8), ("energy", np.float64),
                                               ("forces", np.float64))]
        self._check(self._f("loss_grad")(_i32(B), _p(ap), D, *[_p(k) for k in keep], _p(_c(pred_e, np.float64)),
                                         _p(_c(pred_f, np.float64)), _f64(lambda_e), _f64(lambda_f), _p(bd), _p(ge),
                                         _p(gf)))
        names = ("total", "energy_term", "force_term", "energy_labeled", "force_labeled", "energy_empty",
                 "force_empty")
        return dict(zip(names, bd.tolist())), ge, gf

    # ------------------------------------------------------------ denoise
    def apply_noise(self, pos, Z, sigma, scheme, seed):
        pos, Z = _c(pos, np.float64), _c(Z, np.int32)
        n = len(Z)
        x, lab = np.empty((n, 3)), np.empty((n, 3))
        self._check(self._f("apply_noise")(_i32(n), _p(pos), _p(Z), _f64(sigma), scheme, _u64(seed), _p(x),
                                           _p(lab)))
        return x, lab

    def apply_displacements(self, pos, Z, deltas, scheme):
        pos, Z, d = _c(pos, np.float64), _c(Z, np.int32), _c(deltas, np.float64)
        n = len(Z)
        x, lab = np.empty((n, 3)), np.empty((n, 3))
        self._check(self._f("apply_displacements")(_i32(n), _p(pos), _p(Z), _p(d), scheme, _p(x), _p(lab)))
        return x, lab

    # --------------------------------------------------------- train step
    def train_step(self, cfg, G, B, batch, table, params, rms_v, *, noise_sigma=0.3, noise_scheme=1, seed=0, step=0,
                   lambda_e=1.0, lambda_f=1.0, lr=1e-3, clip=10.0, decay=0.99, eps=1e-8, threads=1):
        H, L, K, rc, D = cfg
        p = _c(params, np.float64).copy()
        v = _c(rms_v, np.float64).copy()
        loss, gn = _f64(), _f64()
        g = np.empty_like(p)
        keep = [_c(batch[k], dt) for k, dt in (("atom_ptr", np.int64), ("pos", np.float64), ("Z", np.int32),
                                               ("dataset_index", np.int32), ("energy_mask", np.uint8),
                                               ("force_mask", np.uint8), ("energy", np.float64),
                                               ("forces", np.float64), ("denoise", np.uint8))]
        args = [H, L, K, _f64(rc), D, G, B, *[_p(k) for k in keep], *self._table_args(table), _f64(noise_sigma),
                noise_scheme, _u64(seed), _i64(step), _f64(lambda_e), _f64(lambda_f), _f64(lr), _f64(clip),
                _f64(decay), _f64(eps), _p(p), _p(v), C.byref(loss), C.byref(gn), _p(g)]
        if self.kind == "ref":
            args.append(threads)
        st = self._f("train_step")(*args)
        if st not in (0, 5):
            self._check(st)
        return dict(params=p, rms_v=v, loss=loss.value, grad_norm=gn.value, grads=g, status=st)

    def worker_step(self, cfg, G, B, g, batch, table, params, *, noise_sigma=0.3, noise_scheme=1, seed=0, step=0,
                    lambda_e=1.0, lambda_f=1.0):
        """Worker g's loss and gradient SUM (port only): one term of the step body."""
        if self.kind != "port":
            raise OracleError("worker_step is provided by the plain-C port only")
        H, L, K, rc, D = cfg
        keep = [_c(batch[k], dt) for k, dt in (("atom_ptr", np.int64), ("pos", np.float64), ("Z", np.int32),
                                               ("dataset_index", np.int32), ("energy_mask", np.uint8),
                                               ("force_mask", np.uint8), ("energy", np.float64),
                                               ("forces", np.float64), ("denoise", np.uint8))]
        loss = _f64()
        g_out = np.empty(self.param_count(cfg))
        self._check(self.lib.lor_worker_step(H, L, K, _f64(rc), D, G, B, g, *[_p(k) for k in keep],
                                             *self._table_args(table), _f64(noise_sigma), noise_scheme, _u64(seed),
                                             _i64(step), _f64(lambda_e), _f64(lambda_f),
                                             _p(_c(params, np.float64)), C.byref(loss), _p(g_out)))
        return loss.value, g_out

    # ---------------------------------------------------------- scheduler
    def greedy_assign(self, atoms, G, B):
        a = _c(atoms, np.int64)
        o = np.empty(len(a), np.int32)
        self._check(self._f("greedy_assign")(_p(a), _i64(len(a)), G, B, _p(o)))
        return o

    _MODES = {"balanced": 0, "greedy_only": 1, "naive": 2}

    def plan(self, atoms, G, B, S, seed, mode="balanced"):
        a = _c(atoms, np.int64)
        n = len(a)
        m = self._MODES[mode]
        if self.kind == "ref":
            h = self.lib.lref_plan(_p(a), _i64(n), G, B, S, _u64(seed), m)
            if not h:
                raise OracleError(self.lib.lref_last_error().decode())
            nb, dr = _i64(), _i64()
            self.lib.lref_plan_info(_P(h), C.byref(nb), C.byref(dr))
            nb, dr = nb.value, dr.value
            tot = nb * G * B
            out = dict(sample=np.empty(tot, np.int64), worker=np.empty(tot, np.int32), atoms=np.empty(tot, np.int64),
                       split=np.empty(tot, np.int64), chunk_rank=np.empty(tot, np.int64),
                       worker_atoms=np.empty(nb * G, np.int64))
            self.lib.lref_plan_copy(_P(h), *[_p(out[k]) for k in ("sample", "worker", "atoms", "split",
                                                                 "chunk_rank", "worker_atoms")])
            mx, mean, mono, grow = _f64(), _f64(), _i64(), _i64()
            self.lib.lref_schedule_metrics(_P(h), C.byref(mx), C.byref(mean), C.byref(mono), C.byref(grow))
            self.lib.lref_plan_free(_P(h))
        else:
            cap = max(n, 1)
            out = dict(sample=np.empty(cap, np.int64), worker=np.empty(cap, np.int32), atoms=np.empty(cap, np.int64),
                       split=np.empty(cap, np.int64), chunk_rank=np.empty(cap, np.int64),
                       worker_atoms=np.empty(cap, np.int64))
            dr = _i64()
            nb = self.lib.lor_plan(_p(a), _i64(n), G, B, S, _u64(seed), m,
                                   *[_p(out[k]) for k in ("sample", "worker", "atoms", "split", "chunk_rank",
                                                          "worker_atoms")], C.byref(dr))
            if nb < 0:
                raise OracleError(self.lib.lor_last_error().decode())
            dr = dr.value
            tot = nb * G * B
            for k in ("sample", "worker", "atoms", "split", "chunk_rank"):
                out[k] = out[k][:tot]
            out["worker_atoms"] = out["worker_atoms"][:nb * G]
            mx, mean, mono, grow = _f64(), _f64(), _i64(), _i64()
            self.lib.lor_schedule_metrics(_i64(nb), G, B, _p(out["worker"]), _p(out["atoms"]), _p(out["split"]),
                                          _p(out["chunk_rank"]), C.byref(mx), C.byref(mean), C.byref(mono),
                                          C.byref(grow))
        out.update(n_batches=nb, dropped=dr, max_imbalance=mx.value, mean_imbalance=mean.value,
                   monotonicity_violations=mono.value, growth_events=grow.value)
        return out

    # ------------------------------------------------------ trace/dataset
    _KINDS = {"constant": 0, "uniform": 1, "lognormal": 2, "bimodal": 3}

    def make_trace(self, kind="lognormal", count=1000, min_atoms=1, max_atoms=300, constant_atoms=15.0, mode=15.0,
                   sigma=0.45, mode_a=15.0, sigma_a=0.30, mode_b=160.0, sigma_b=0.30, weight_a=0.5, seed=0):
        o = np.empty(count, np.int64)
        self._check(self._f("make_trace")(self._KINDS[kind], _i64(count), _i64(min_atoms), _i64(max_atoms),
                                          _f64(constant_atoms), _f64(mode), _f64(sigma), _f64(mode_a),
                                          _f64(sigma_a), _f64(mode_b), _f64(sigma_b), _f64(weight_a), _u64(seed),
                                          _p(o)))
        return o

    def temperature_counts(self, sizes, T):
        s = _c(sizes, np.float64)
        o = np.empty(len(s))
        self._check(self._f("temperature_counts")(_p(s), len(s), _f64(T), _p(o)))
        return o

    def build_epoch_index(self, repeats, sizes, seed):
        r, s = _c(repeats, np.float64), _c(sizes, np.int64)
        cap = int(sum(int(np.rint(x)) for x in r)) + 8
        osub, osam = np.empty(cap, np.int32), np.empty(cap, np.int64)
        n = self._f("build_epoch_index")(_p(r), _p(s), len(s), _u64(seed), _i64(cap), _p(osub), _p(osam))
        if n < 0:
            raise OracleError(self._f("last_error")().decode())
        return osub[:n], osam[:n]

    _TASKS = {"energy_and_forces": 0, "energy_only": 1, "denoising": 2}

    def synth_generate(self, count, seed, *, task="energy_and_forces", mode=15.0, sigma=0.45, min_atoms=2,
                       max_atoms=300, elements=(6,), relax_steps=6, relax_step=0.02, energy_scale=1.0,
                       offsets=None):
        el = _c(list(elements), np.int32)
        offsets = offsets or {}
        oz = _c(list(offsets.keys()) or [0], np.int32)
        ov = _c(list(offsets.values()) or [0.0], np.float64)
        t = self._TASKS[task]
        if self.kind == "ref":
            h = self.lib.lref_synth_generate(t, _i64(count), _f64(mode), _f64(sigma), min_atoms, max_atoms, _p(el),
                                             len(el), relax_steps, _f64(relax_step), _f64(energy_scale), _p(oz),
                                             _p(ov), len(offsets), _u64(seed))
            if not h:
                raise OracleError(self.lib.lref_last_error().decode())
            cnt, tot = _i64(), _i64()
            self.lib.lref_samples_info(_P(h), C.byref(cnt), C.byref(tot))
            B, N = cnt.value, tot.value
            ap = np.empty(B + 1, np.int64)
        else:
            B = count
            ap = np.empty(B + 1, np.int64)
            self.lib.lor_synth_counts(_i64(count), _f64(mode), _f64(sigma), min_atoms, max_atoms, _u64(seed), _p(ap))
            N = int(ap[-1])
        b = dict(atom_ptr=ap, pos=np.empty((N, 3)), Z=np.empty(N, np.int32), energy_mask=np.empty(B, np.uint8),
                 force_mask=np.empty(B, np.uint8), energy=np.empty(B), forces=np.empty((N, 3)))
        if self.kind == "ref":
            self.lib.lref_samples_copy(_P(h), _p(ap), _p(b["pos"]), _p(b["Z"]), _p(b["energy_mask"]),
                                       _p(b["force_mask"]), _p(b["energy"]), _p(b["forces"]))
            self.lib.lref_samples_free(_P(h))
        else:
            self.lib.lor_synth_fill(t, _i64(count), _f64(mode), _f64(sigma), min_atoms, max_atoms, _p(el), len(el),
                                    relax_steps, _f64(relax_step), _f64(energy_scale), _p(oz), _p(ov), len(offsets),
                                    _u64(seed), _p(ap), _p(b["pos"]), _p(b["Z"]), _p(b["energy_mask"]),
                                    _p(b["force_mask"]), _p(b["energy"]), _p(b["forces"]))
        b["dataset_index"] = np.zeros(B, np.int32)
        b["denoise"] = np.full(B, 1 if task == "denoising" else 0, np.uint8)
        return b


_cache: dict = {}


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref() -> OracleLib:
    if "ref" not in _cache:
        _cache["ref"] = OracleLib(REF_PATH, "ref")
    return _cache["ref"]


def port() -> OracleLib:
    if "port" not in _cache:
        _cache["port"] = OracleLib(PORT_PATH, "port")
    return _cache["port"]
