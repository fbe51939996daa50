/*
 * oracle/lamm_oracle.h - plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see lamm_oracle.c). Only tests/, __graft_entry__
 * smoke() and bench.py's cpu_baseline leg may load the built library.
 *
 * Packed-batch conventions are the ones documented in oracle/ref_capi.cpp and
 * include/lamm_b200.h; every function mirrors an lref_* entry point of
 * oracle/_ref so the two can be compared bit for bit.
 */
#ifndef LAMM_ORACLE_H
#define LAMM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t lor_mix_seed(uint64_t a, uint64_t b);
void lor_rng_normals(uint64_t seed, int64_t n, double* out);
void lor_rng_uniforms(uint64_t seed, int64_t n, double* out);
void lor_rng_u64(uint64_t seed, int64_t n, uint64_t* out);
void lor_rng_bounded(uint64_t seed, int64_t n, uint64_t bound, uint64_t* out);
void lor_rng_permutation(uint64_t seed, int64_t n, int64_t* out);

/* Periodic cells for the batch calls that follow ([B][3][3] rows = lattice
 * vectors, all-zero rows block = non-periodic sample; cellinv its inverse), or
 * NULL. Minimum image; parity-unpinned extension (the reference has no cells). */
void lor_set_cells(const double* cells, const double* cellinv);
/* Per-axis periodicity [B][3] of the cells above (NULL: all periodic). */
void lor_set_pbc(const uint8_t* pbc);
/* Image range m[k] of a cell (see lamm_oracle.c; -1 = non-periodic axis). */
void lor_image_range(const double* cellinv, const uint8_t* pbc, double cutoff, int* m);
int lor_cell_inverse(const double* cell, double* out);
int64_t lor_neighbor_list(int32_t n, const double* pos, const int32_t* Z, double cutoff, int64_t cap,
                          int32_t* oi, int32_t* oj, double* odist, double* ounit);

int64_t lor_param_count(int H, int L, int K, int D);
int lor_init_params(int H, int L, int K, double rc, int D, uint64_t seed, double* out);
int lor_forward(int H, int L, int K, double rc, int D, const double* params, int32_t B, const int64_t* atom_ptr,
                const double* pos, const int32_t* Z, double* out_energy, double* out_forces);
int lor_forward_cache(int H, int L, int K, double rc, int D, const double* params, int32_t n, const double* pos,
                      const int32_t* Z, double* h_all, double* mt_all);
int lor_backward(int H, int L, int K, double rc, int D, const double* params, int32_t B, const int64_t* atom_ptr,
                 const double* pos, const int32_t* Z, const double* up_energy, const double* up_forces,
                 double* grads_accum);

int lor_normalize_labels(int32_t B, const int64_t* atom_ptr, const double* pos, const int32_t* Z,
                         const int32_t* dsidx, const uint8_t* emask, const uint8_t* fmask, const double* energy,
                         const double* forces, int ntab, const double* rho, const uint8_t* rho_has,
                         const double* mean, const double* stdv, const double* fstd, const uint8_t* has,
                         double* out_energy, double* out_forces);
int lor_loss_grad(int32_t B, const int64_t* atom_ptr, int D, const int32_t* dsidx, const uint8_t* emask,
                  const uint8_t* fmask, const double* energy, const double* forces, const double* pred_energy,
                  const double* pred_forces, double lambda_e, double lambda_f, double* breakdown, double* g_energy,
                  double* g_forces);

int lor_apply_noise(int32_t n, const double* pos, const int32_t* Z, double sigma, int scheme, uint64_t seed,
                    double* noisy, double* labels);
int lor_apply_displacements(int32_t n, const double* pos, const int32_t* Z, const double* deltas, int scheme,
                            double* noisy, double* labels);

int lor_train_step(int H, int L, int K, double rc, int D, int G, int B, const int64_t* atom_ptr, const double* pos,
                   const int32_t* Z, const int32_t* dsidx, const uint8_t* emask, const uint8_t* fmask,
                   const double* energy, const double* forces, const uint8_t* denoise_flag, int ntab,
                   const double* rho, const uint8_t* rho_has, const double* mean, const double* stdv,
                   const double* fstd, const uint8_t* has, double noise_sigma, int noise_scheme, uint64_t seed,
                   int64_t step, double lambda_e, double lambda_f, double lr, double clip, double decay, double eps,
                   double* params, double* rms_v, double* out_loss, double* out_grad_norm, double* out_grads);

int lor_worker_step(int H, int L, int K, double rc, int D, int G, int B, int g, const int64_t* atom_ptr,
                    const double* pos, const int32_t* Z, const int32_t* dsidx, const uint8_t* emask,
                    const uint8_t* fmask, const double* energy, const double* forces, const uint8_t* denoise_flag,
                    int ntab, const double* rho, const uint8_t* rho_has, const double* mean, const double* stdv,
                    const double* fstd, const uint8_t* has, double noise_sigma, int noise_scheme, uint64_t seed,
                    int64_t step, double lambda_e, double lambda_f, const double* params, double* out_loss,
                    double* out_grads);

int lor_greedy_assign(const int64_t* atoms, int64_t n, int G, int B, int32_t* out);
/* Returns the number of mini-batches (or < 0 on error). All outputs have
 * capacity n (scheduled samples never exceed n). */
int64_t lor_plan(const int64_t* atoms, int64_t n, int G, int B, int S, uint64_t seed, int mode, int64_t* sample,
                 int32_t* worker, int64_t* oatoms, int64_t* split, int64_t* chunk_rank, int64_t* worker_atoms,
                 int64_t* dropped);
void lor_schedule_metrics(int64_t nbatches, int G, int B, const int32_t* worker, const int64_t* atoms,
                          const int64_t* split, const int64_t* chunk_rank, double* max_imb, double* mean_imb,
                          int64_t* mono, int64_t* growth);

int lor_make_trace(int kind, int64_t count, int64_t min_atoms, int64_t max_atoms, double constant_atoms,
                   double mode, double sigma, double mode_a, double sigma_a, double mode_b, double sigma_b,
                   double weight_a, uint64_t seed, int64_t* out);
int lor_temperature_counts(const double* sizes, int k, double T, double* out);
int64_t lor_build_epoch_index(const double* repeats, const int64_t* sizes, int k, uint64_t seed, int64_t cap,
                              int32_t* out_subset, int64_t* out_sample);

/* Synthetic Morse clusters (S/dataset.cpp:161-247): the per-sample atom counts
 * come first (lor_synth_counts), then the packed samples (lor_synth_fill). */
int lor_synth_counts(int64_t count, double mode, double sigma, int min_atoms, int max_atoms, uint64_t seed,
                     int64_t* atom_ptr);
int lor_synth_fill(int task, int64_t count, double mode, double sigma, int min_atoms, int max_atoms,
                   const int32_t* elements, int nelem, int relax_steps, double relax_step, double energy_scale,
                   const int32_t* off_z, const double* off_v, int noff, uint64_t seed, const int64_t* atom_ptr,
                   double* pos, int32_t* Z, uint8_t* emask, uint8_t* fmask, double* energy, double* forces);

const char* lor_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
