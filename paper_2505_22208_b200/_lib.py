"""Loader for liblamm_b200.so (the C ABI in include/lamm_b200.h).

The library is built in-tree by ``make -C paper_2505_22208_b200/csrc`` (or
``__graft_entry__.build()``). There is no fallback: if the shared object is
missing or fails to load, importing the API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblamm_b200.so")


class LammError(RuntimeError):
    """LAMM_EINTERNAL / LAMM_ECUDA / LAMM_ENCCL."""


class InputError(ValueError):
    """LAMM_EINPUT — the reference's lamm::InputError (H/core.hpp:22-26)."""


class NonFiniteError(RuntimeError):
    """LAMM_ENONFINITE — non-finite loss or gradient (S/trainer.cpp:322-324)."""


class ModelConfigC(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("layers", C.c_int32), ("rbf", C.c_int32), ("heads", C.c_int32),
                ("cutoff", C.c_double)]


class BatchViewC(C.Structure):
    _fields_ = [("n_samples", C.c_int32), ("n_atoms", C.c_int64), ("atom_ptr", C.c_void_p),
                ("positions", C.c_void_p), ("atomic_numbers", C.c_void_p), ("dataset_index", C.c_void_p),
                ("energy_mask", C.c_void_p), ("force_mask", C.c_void_p), ("energy", C.c_void_p),
                ("forces", C.c_void_p), ("denoise", C.c_void_p), ("cell", C.c_void_p), ("pbc", C.c_void_p)]


class NormalizerC(C.Structure):
    _fields_ = [("rho", C.c_double * 119), ("rho_has", C.c_uint8 * 119), ("energy_mean", C.c_double),
                ("energy_std", C.c_double), ("force_std", C.c_double), ("has_energy_stats", C.c_uint8)]


class SimCostC(C.Structure):
    _fields_ = [("alpha_s", C.c_double), ("beta_s_per_atom", C.c_double), ("gamma_s", C.c_double),
                ("delta_s", C.c_double)]


class SimTotalsC(C.Structure):
    _fields_ = [("total_s", C.c_double), ("throughput_samples_per_s", C.c_double), ("realloc_events", C.c_int64),
                ("samples", C.c_int64)]


class CostModelC(C.Structure):
    _fields_ = [("per_sample", C.c_double), ("per_atom", C.c_double), ("per_edge", C.c_double)]


class RefTableC(C.Structure):
    _fields_ = [("n_tables", C.c_int32), ("rho", C.c_void_p), ("rho_has", C.c_void_p),
                ("energy_mean", C.c_void_p), ("energy_std", C.c_void_p), ("force_std", C.c_void_p),
                ("has_energy_stats", C.c_void_p)]


class LossConfigC(C.Structure):
    _fields_ = [("lambda_energy", C.c_double), ("lambda_force", C.c_double)]


class LossBreakdownC(C.Structure):
    _fields_ = [("total", C.c_double), ("energy_term", C.c_double), ("force_term", C.c_double),
                ("energy_labeled", C.c_int32), ("force_labeled", C.c_int32), ("energy_empty", C.c_int32),
                ("force_empty", C.c_int32)]


class TrainConfigC(C.Structure):
    _fields_ = [("learning_rate", C.c_double), ("clip_norm", C.c_double), ("rms_decay", C.c_double),
                ("rms_epsilon", C.c_double), ("noise_sigma", C.c_double), ("noise_scheme", C.c_int32),
                ("seed", C.c_uint64), ("lambda_energy", C.c_double), ("lambda_force", C.c_double)]


class StepResultC(C.Structure):
    _fields_ = [("loss", C.c_double), ("grad_norm", C.c_double), ("local", LossBreakdownC),
                ("n_atoms", C.c_int64), ("n_edges", C.c_int64), ("status", C.c_int32), ("retries", C.c_int32),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64)]


class EvalResultC(C.Structure):
    _fields_ = [("energy_mae", C.c_double), ("force_mae", C.c_double), ("energy_count", C.c_int64),
                ("force_count", C.c_int64)]


# Every symbol include/lamm_b200.h declares (tests check the export table).
EXPORTS = [
    "lamm_last_error", "lamm_ctx_create", "lamm_ctx_destroy", "lamm_ctx_set_option", "lamm_param_count",
    "lamm_init_params", "lamm_params_set", "lamm_params_get", "lamm_rms_state_set", "lamm_rms_state_get",
    "lamm_batch_set", "lamm_ref_table_set", "lamm_labels_get", "lamm_neighbor_list", "lamm_neighbor_list_copy",
    "lamm_forward", "lamm_forward_cache_get", "lamm_loss_grad", "lamm_backward", "lamm_comm_unique_id",
    "lamm_comm_init", "lamm_train_step", "lamm_optimizer_step", "lamm_grads_get", "lamm_sync",
    "lamm_event_record", "lamm_event_elapsed_ms", "lamm_kernel_times", "lamm_kernel_times_reset",
    "lamm_last_step_launches", "lamm_greedy_assign", "lamm_plan", "lamm_schedule_metrics", "lamm_make_trace",
    "lamm_temperature_counts", "lamm_build_epoch_index", "lamm_synth_counts", "lamm_synth_fill",
    "lamm_mix_seed", "lamm_rng_normals", "lamm_stage", "lamm_train_step_staged", "lamm_anomalies",
    "lamm_train_step_submit", "lamm_train_step_wait",
    "lamm_flush_l2", "lamm_step_times", "lamm_evaluate", "lamm_cell_inverse",
    "lamm_checkpoint_save", "lamm_checkpoint_load", "lamm_rms_state_save", "lamm_rms_state_load",
    "lamm_subset_info", "lamm_subset_read", "lamm_train_step_workers", "lamm_ctx_get_info",
    "lamm_sample_cost", "lamm_plan_cost", "lamm_filter_max_atoms", "lamm_split_train_val", "lamm_apply_noise",
    "lamm_pseudo_force_std", "lamm_fit_normalizer", "lamm_init_heads", "lamm_last_step_compute_ms",
    "lamm_train_step_staged_next", "lamm_simulate",
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `make -C paper_2505_22208_b200/csrc` "
                              "(or __graft_entry__.build()) — there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        L.lamm_last_error.restype = C.c_char_p
        L.lamm_param_count.restype = C.c_int64
        L.lamm_param_count.argtypes = [C.POINTER(ModelConfigC)]
        L.lamm_mix_seed.restype = C.c_uint64
        L.lamm_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.lamm_last_step_launches.restype = C.c_int64
        L.lamm_anomalies.restype = C.c_int64
        L.lamm_ctx_destroy.restype = None
        L.lamm_ctx_create.argtypes = [C.c_int, C.POINTER(ModelConfigC), C.POINTER(C.c_void_p)]
        for fn in ("lamm_ctx_destroy",):
            getattr(L, fn).argtypes = [C.c_void_p]
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().lamm_last_error().decode(errors="replace")
    if status == 1:
        raise InputError(msg)
    if status == 5:
        raise NonFiniteError(msg)
    raise LammError(f"status {status}: {msg}")
