"""B200-native LaMM load-balanced energy/force train step.

A drop-in for the reference's (arXiv 2505.22208, /root/reference/proj/core)
data-parallel train-step path: liblamm_b200.so (C ABI, include/lamm_b200.h)
with hand-written sm_100a CUDA kernels, host C++ for the atom-count load
balancer, and NCCL for the one gradient allreduce per step. This package is
the host-side mirror of the reference API; there is no CPU compute fallback.
"""
from .api import (Device, LossConfig, ModelConfig, TrainConfig, build_epoch_index, cell_inverse, comm_unique_id,  # noqa: F401
                  concat, empty_table, greedy_assign, init_params, make_trace, mix_seed, param_count, plan,
                  rng_normals, select, synth_generate, temperature_counts, CostModel, sample_cost, plan_cost,
                  fit_cost_model, filter_max_atoms, split_train_val, apply_noise, pseudo_force_std,
                  fit_normalizer, init_heads, simulate)
from ._lib import InputError, LammError, NonFiniteError, LIB_PATH  # noqa: F401
