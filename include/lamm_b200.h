/*
 * lamm_b200.h - C ABI of the B200-native LaMM hot path (liblamm_b200.so).
 *
 * Drop-in boundary for the load-balanced energy/force train step of the LaMM
 * reference C++ core (/root/reference/proj/core, namespace lamm). The reference
 * has no plugin registry or FFI: its boundary is the C++ API of lamm::core. Each
 * entry point below names the reference function it replaces (H = include/lamm,
 * S = src). Conventions:
 *
 *   - extern "C", plain pointers and sizes, no exceptions cross the boundary.
 *   - Every call returns a lamm_status; lamm_last_error() holds the message
 *     (thread-local). LAMM_EINPUT corresponds to the reference's InputError
 *     (H/core.hpp:22-26, CLI exit 1); LAMM_ENONFINITE to the runtime_error of
 *     S/trainer.cpp:322-324.
 *   - One lamm_ctx per GPU, bound to one CUDA stream, driven by one host thread.
 *     Views are non-owning; the ctx owns device buffers sized to the high-water
 *     mark and grown geometrically.
 *   - Packed batch layout (CSR over atoms):
 *       atom_ptr[B+1] int64, positions[3N] f64 (atom-major xyz, Angstrom),
 *       atomic_numbers[N] int32 in [1,118], dataset_index[B] int32 (head d),
 *       energy_mask[B]/force_mask[B] uint8 (m_E, m_F), energy[B] f64,
 *       forces[3N] f64 (rows of force-labelled samples; ignored otherwise),
 *       denoise[B] uint8 (nullable: sample comes from a denoising subset and
 *       gets labels from make_denoising_sample, S/denoise.cpp:42-53),
 *       cell[B][3][3] f64 (nullable: periodic cells, minimum image).
 *   - Parameters: fp64, flat, for_each_tensor order (H/model.hpp:59-66):
 *       embedding 118xH, filter[L] HxK, update[L] HxH, energy_head HxD,
 *       force_head (2H+K)xD, each row-major.
 *   - Predictions use the reference layout per sample (H/model.hpp:99-108):
 *       energy[B*D]; forces: block at 3*D*atom_ptr[s], inside it (d*n+j)*3+c.
 */
#ifndef LAMM_B200_H
#define LAMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LAMM_OK = 0,
    LAMM_EINPUT = 1,     /* invalid input (reference InputError) */
    LAMM_EINTERNAL = 2,  /* any other failure */
    LAMM_ECUDA = 3,      /* CUDA runtime error */
    LAMM_ENCCL = 4,      /* NCCL error */
    LAMM_ENONFINITE = 5  /* non-finite loss or gradient (S/trainer.cpp:322-324) */
} lamm_status;

typedef struct lamm_ctx lamm_ctx;

/* lamm::model::ModelConfig, H/model.hpp:34-40. The sm_100a kernels are
 * instantiated for (hidden, rbf) in {(128,16), (128,8), (64,16), (64,8), (32,8), (32,16)}; layers <= 8,
 * heads <= 16. */
typedef struct {
    int32_t hidden;
    int32_t layers;
    int32_t rbf;
    int32_t heads;
    double cutoff;
} lamm_model_config;

typedef struct {
    int32_t n_samples;
    int64_t n_atoms;
    const int64_t* atom_ptr;
    const double* positions;
    const int32_t* atomic_numbers;
    const int32_t* dataset_index;
    const uint8_t* energy_mask;
    const uint8_t* force_mask;
    const double* energy;
    const double* forces;
    const uint8_t* denoise;
    /* Periodic cells (extension; the reference has none): [n_samples][3][3], row k =
     * lattice vector k (Angstrom); an all-zero cell marks a non-periodic sample.
     * NULL: every sample is non-periodic (the reference's behaviour, bit-exact).
     * A periodic sample's pairs are (i, j, n): every image of j within the cutoff,
     * n the integer shift relative to j's minimum image (cells at least 2 * cutoff
     * wide on every periodic axis: exactly the minimum image; narrower cells:
     * several images per pair and self-images (i, i, n != 0)); order i-major, j
     * ascending, n lexicographic (oracle/lamm_oracle.c states the fp64 sequence).
     * More than 4096 images per pair (cells far below the cutoff) is LAMM_EINPUT. */
    const double* cell;
    /* Per-axis periodicity of the cells, [n_samples][3] (1 periodic, 0 open: no
     * wrapping along lattice vector k, e.g. slabs {1, 1, 0}). NULL: all periodic.
     * Ignored for non-periodic samples. */
    const uint8_t* pbc;
} lamm_batch_view;

/* lamm::loss::ReferenceTable / DatasetNormalizer, H/loss.hpp:31-44. rho and
 * rho_has are [n_tables][119] indexed by Z (rho_has stands in for std::map key
 * presence). */
typedef struct {
    int32_t n_tables;
    const double* rho;
    const uint8_t* rho_has;
    const double* energy_mean;
    const double* energy_std;
    const double* force_std;
    const uint8_t* has_energy_stats;
} lamm_ref_table;

/* lamm::loss::LossConfig, H/loss.hpp:26-29 */
typedef struct {
    double lambda_energy;
    double lambda_force;
} lamm_loss_config;

/* lamm::loss::LossBreakdown, H/loss.hpp:62-70 */
typedef struct {
    double total;
    double energy_term;
    double force_term;
    int32_t energy_labeled;
    int32_t force_labeled;
    int32_t energy_empty;
    int32_t force_empty;
} lamm_loss_breakdown;

/* The step-body subset of lamm::trainer::TrainConfig (H/trainer.hpp:33-50). */
typedef struct {
    double learning_rate;  /* 1e-3 */
    double clip_norm;      /* 10   */
    double rms_decay;      /* 0.99 */
    double rms_epsilon;    /* 1e-8 */
    double noise_sigma;    /* 0.3 Angstrom */
    int32_t noise_scheme;  /* 1 = centered, 0 = baseline (H/denoise.hpp:19) */
    uint64_t seed;         /* TrainConfig.seed: denoise streams derive from it */
    double lambda_energy;  /* 1 */
    double lambda_force;   /* 1 */
} lamm_train_config;

typedef struct {
    double loss;          /* sum over ranks of per-rank Eq.(5) loss, / G (S/trainer.cpp:320) */
    double grad_norm;     /* ||mean gradient|| before clipping (S/trainer.cpp:321) */
    lamm_loss_breakdown local; /* this rank's masked_loss_grad breakdown */
    int64_t n_atoms;      /* atoms in this rank's device-batch */
    int64_t n_edges;      /* directed pairs built for it */
    int32_t status;       /* lamm_status of the step */
    int32_t retries;      /* edge-capacity regrowth re-runs */
    int64_t h2d_bytes;    /* bytes copied host -> device for this step */
    int64_t d2h_bytes;    /* bytes copied device -> host for this step's result */
} lamm_step_result;

/* ------------------------------------------------------------ context --- */
const char* lamm_last_error(void);
int lamm_ctx_create(int device, const lamm_model_config* cfg, lamm_ctx** out);
void lamm_ctx_destroy(lamm_ctx* ctx);
/* Options: "graph" (CUDA-graph capture of the step, default 1),
 * "profile" (per-kernel CUDA events inside the step, default 0),
 * "export_fp64" (keep fp64 pair distance/unit for lamm_neighbor_list_copy),
 * "pdl" (programmatic dependent launch between the step's kernels, default 1),
 * "rank_local" (default 0: a train step with workers > 1 on a context without
 * a communicator is refused; 1: run and apply this rank's share alone, for
 * per-rank timing and per-rank gradient checks). */
int lamm_ctx_set_option(lamm_ctx* ctx, const char* name, int64_t value);

/* ---------------------------------------------------------- parameters --- */
int64_t lamm_param_count(const lamm_model_config* cfg);
/* lamm::model::init_params, H/model.hpp:72 (host, bit-exact with the reference). */
int lamm_init_params(const lamm_model_config* cfg, uint64_t seed, double* out);
int lamm_params_set(lamm_ctx* ctx, const double* flat, size_t n);
int lamm_params_get(lamm_ctx* ctx, double* flat, size_t n);
/* RMS optimizer state v (S/trainer.cpp:29-35), same layout as the params. */
int lamm_rms_state_set(lamm_ctx* ctx, const double* flat, size_t n);
int lamm_rms_state_get(lamm_ctx* ctx, double* flat, size_t n);

/* --------------------------------------------------------------- batch --- */
/* Uploads a device-batch (H2D) and prepares it on the device. Labels are taken
 * as given (already normalized) unless lamm_ref_table_set installed a table, in
 * which case normalize_labels (S/loss.cpp:113-126) runs on the device. */
int lamm_batch_set(lamm_ctx* ctx, const lamm_batch_view* batch);
int lamm_ref_table_set(lamm_ctx* ctx, const lamm_ref_table* table); /* NULL clears */
/* Normalized labels of the current batch (device -> host), for parity checks. */
int lamm_labels_get(lamm_ctx* ctx, double* energy, double* forces);

/* build_neighbor_list (H/core.hpp:83, S/core.cpp:30-48) for every sample of the
 * current batch, bit-exact pair set and order (i-major, j ascending, local
 * indices). Returns the pair count in *n_pairs. */
int lamm_neighbor_list(lamm_ctx* ctx, int64_t* n_pairs);
/* Copies the list: sample_pair_ptr[B+1]; i, j local to the sample; dist and
 * unit[3] are fp64 and bit-identical to the reference when "export_fp64" is set. */
int lamm_neighbor_list_copy(lamm_ctx* ctx, int64_t* sample_pair_ptr, int32_t* i, int32_t* j, double* dist,
                            double* unit);

/* lamm::model::forward (H/model.hpp:123-124) over the batch; the ForwardCache
 * stays on the device. energy/forces are nullable (leave on device). */
int lamm_forward(lamm_ctx* ctx, double* energy, double* forces);
/* ForwardCache rows of one layer (debug/parity): which = 0 -> h[l] (l in 0..L),
 * 1 -> tanh(m)[l] (l in 0..L-1); out is [N][H] fp64. */
int lamm_forward_cache_get(lamm_ctx* ctx, int which, int layer, double* out);

/* lamm::loss::masked_loss_grad (H/loss.hpp:81-84) on the forward predictions
 * and the batch labels; keeps d(loss)/d(prediction) on the device. g_energy
 * [B*D] and g_forces (prediction layout) are nullable copies. */
int lamm_loss_grad(lamm_ctx* ctx, const lamm_loss_config* cfg, lamm_loss_breakdown* out, double* g_energy,
                   double* g_forces);

/* lamm::model::backward (H/model.hpp:128-129): parameter gradients of the
 * batch. Upstream gradients come from up_energy/up_forces when given (prediction
 * layout), else from the last lamm_loss_grad. Accumulate semantics: when
 * grads_accum is non-NULL the batch gradient is ADDED into it (fp64, flat). */
int lamm_backward(lamm_ctx* ctx, const double* up_energy, const double* up_forces, double* grads_accum);

/* trainer::EvalResult, H/trainer.hpp:129-134 */
typedef struct {
    double energy_mae;    /* meV per atom over energy-labelled samples, NaN if none */
    double force_mae;     /* meV/Angstrom over force-labelled samples, NaN if none */
    int64_t energy_count;
    int64_t force_count;
} lamm_eval_result;

/* lamm::trainer::evaluate (H/trainer.hpp:143-144, S/trainer.cpp:528-553): the
 * current parameters on `batch` (raw labels, no denoising), each sample's own
 * head denormalized with the installed reference table, physical-unit MAEs.
 * Replaces the context's current batch. */
int lamm_evaluate(lamm_ctx* ctx, const lamm_batch_view* batch, lamm_eval_result* out);

/* ----------------------------------------------------------- train step --- */
/* NCCL communicator for data parallelism over `nranks` GPUs (one ctx per GPU,
 * one process per GPU). unique_id is the 128-byte ncclUniqueId from rank 0. */
int lamm_comm_unique_id(void* out128);
int lamm_comm_init(lamm_ctx* ctx, int nranks, int rank, const void* unique_id128);

/* One optimizer step of the LaMM train loop, semantics of S/trainer.cpp:258-327
 * for rank `rank` of `workers`: `batch` holds this rank's B scheduled samples
 * (MiniBatch.samples[rank*B .. rank*B+B), S/scheduler.cpp:43-58). Runs
 * denoise -> normalize -> neighbour list -> forward -> per-rank masked loss ->
 * backward -> one NCCL allreduce of the packed gradient -> /G -> norm ->
 * clip -> RMS step, all on the device (CUDA graph). Denoising draws use the
 * reference stream mix_seed(mix_seed(seed, 0x4e4f4953 + step), rank*B + b). */
int lamm_train_step(lamm_ctx* ctx, const lamm_batch_view* batch, const lamm_train_config* cfg, int64_t step,
                    int32_t workers, int32_t rank, lamm_step_result* result);

/* The same step for `workers` SIMULATED workers on this one device, the
 * reference's own semantics (S/trainer.cpp:262-319): batches[g] holds worker
 * g's B samples; each worker's denoise -> forward -> masked loss -> backward
 * runs in worker order, the gradients and loss terms are summed in fp64, then
 * /G -> norm -> clip -> RMS step. result->n_atoms/n_edges are totals over the
 * workers, result->local is the last worker's breakdown. Needs a context
 * without a communicator. */
int lamm_train_step_workers(lamm_ctx* ctx, const lamm_batch_view* batches, int32_t workers,
                            const lamm_train_config* cfg, int64_t step, lamm_step_result* result);

/* Pipelined train steps (the step body of S/trainer.cpp:258-327, same results as
 * lamm_train_step in the same order): lamm_train_step_submit packs the batch into
 * one of two pinned host blobs and enqueues upload -> step -> optimizer -> header
 * read-back without waiting, so the host packs step k+1 while the device runs
 * step k; lamm_train_step_wait(ticket) waits for the oldest outstanding step and
 * fills its result. At most two steps in flight; tickets are waited for in
 * order. A step that overflows the edge capacity (or runs non-finite) makes the
 * steps behind it skip their update on the device; the wait then reruns the
 * chain in order, so parameters and results equal the synchronous sequence
 * (a non-finite step still reports LAMM_ENONFINITE at its wait). The synchronous
 * step calls are refused while tickets are outstanding. */
int lamm_train_step_submit(lamm_ctx* ctx, const lamm_batch_view* batch, const lamm_train_config* cfg, int64_t step,
                           int32_t workers, int32_t rank, int64_t* ticket);
int lamm_train_step_wait(lamm_ctx* ctx, int64_t ticket, lamm_step_result* result);

/* Device-resident staging for throughput runs: packs a device-batch exactly as
 * lamm_train_step would (denoise draws for `step`, `rank`) into HBM slot
 * `slot` (0..1023); lamm_train_step_staged then runs the same step from that
 * slot (device-to-device copy + graph) with no host work. sync = 0 returns
 * without waiting (result may be NULL); errors are then counted on the device
 * and reported by lamm_anomalies. */
int lamm_stage(lamm_ctx* ctx, const lamm_batch_view* batch, const lamm_train_config* cfg, int64_t step,
               int32_t workers, int32_t rank, int32_t slot);
int lamm_train_step_staged(lamm_ctx* ctx, int32_t slot, int32_t sync, lamm_step_result* result);
/* lamm_train_step_staged with the next step's batch preparation pipelined: the
 * denoise / label / neighbour-list kernels of `next_slot` (independent of the
 * parameters) run on a side stream into a second copy of the batch state while
 * this step's forward/backward/optimizer run; the next call with slot ==
 * next_slot starts directly with its model. next_slot < 0: no prefetch. Results
 * are bit-identical to lamm_train_step_staged; the step's device time (step_ev)
 * includes the prefetch it overlaps. Needs graph capture (options graph 1,
 * profile 0). Any other call first finishes and discards a pending prefetch. */
int lamm_train_step_staged_next(lamm_ctx* ctx, int32_t slot, int32_t next_slot, int32_t sync,
                                lamm_step_result* result);
/* Steps since context creation whose update was skipped (non-finite or edge
 * capacity overflow). */
int64_t lamm_anomalies(lamm_ctx* ctx);
/* Writes `bytes` of scratch on the ctx stream to evict L2 between timed steps. */
int lamm_flush_l2(lamm_ctx* ctx, int64_t bytes);

/* RmsOptimizer::step (S/trainer.cpp:37-53) after scale/norm/clip
 * (S/trainer.cpp:319-326) applied to a host fp64 worker-summed gradient. */
int lamm_optimizer_step(lamm_ctx* ctx, const double* grad_sum, int32_t workers, const lamm_train_config* cfg,
                        double* grad_norm);
/* With a communicator: device time of the last synced step from its upload to the
 * gradient allreduce (this rank's own work; max/mean over ranks = the per-rank
 * step-time imbalance). */
int lamm_last_step_compute_ms(lamm_ctx* ctx, double* ms);
/* Device gradient of the last step (sum over ranks - or over the simulated workers of
 * lamm_train_step_workers, fp64 - before /G), fp64 copy. */
int lamm_grads_get(lamm_ctx* ctx, double* flat, size_t n);

/* ------------------------------------------------------------- timing --- */
int lamm_sync(lamm_ctx* ctx);
/* CUDA events on the ctx stream: record into slot (0..63), elapsed slot a->b. */
int lamm_event_record(lamm_ctx* ctx, int slot);
int lamm_event_elapsed_ms(lamm_ctx* ctx, int slot_a, int slot_b, float* ms);
/* Per-kernel device time accumulated while "profile" is on: names and ms. */
int lamm_kernel_times(lamm_ctx* ctx, int max_kernels, const char** names, double* total_ms, int64_t* launches,
                      int* n_kernels);
int lamm_kernel_times_reset(lamm_ctx* ctx);
/* Device time of every synced train step since the last reset, from CUDA events
 * on the ctx stream around upload -> step -> optimizer (the result D2H and any
 * host work excluded). Reset by lamm_kernel_times_reset. */
int lamm_step_times(lamm_ctx* ctx, double* total_ms, int64_t* steps);
/* Number of this library's kernel launches issued by the last train step. */
int64_t lamm_last_step_launches(lamm_ctx* ctx);
/* Launch geometry of the context, for tests and benchmarks: "grid_edge" (CTAs of
 * the edge kernels), "parts_per_cta" (edge partitions per CTA), "chunk_edges"
 * (edges per TMA-staged chunk), "message_groups" / "edge_groups" / "force_groups"
 * (edge streams per CTA), "message_block" / "edge_block" (edges per walk block),
 * "sm_count", "edge_capacity". Unknown names are LAMM_EINPUT. */
int lamm_ctx_get_info(lamm_ctx* ctx, const char* name, int64_t* value);

/* -------------------------------------------------- host: scheduling --- */
/* lamm::scheduler::greedy_assign, H/scheduler.hpp:66-67 / S/scheduler.cpp:62-89. */
int lamm_greedy_assign(const int64_t* atoms, int64_t n, int32_t workers, int32_t batch_per_worker,
                       int32_t* worker_out);
/* lamm::scheduler::plan (H/scheduler.hpp:74; S/scheduler.cpp:91-203).
 * mode: 0 balanced, 1 greedy_only, 2 naive. Outputs have capacity n; returns
 * the number of mini-batches in *n_batches. Flat ScheduledSample arrays in
 * step-major, worker-major order; worker_atoms[n_batches*workers]. */
int lamm_plan(const int64_t* atoms, int64_t n, int32_t workers, int32_t batch_per_worker, int32_t num_splits,
              uint64_t seed, int32_t mode, int64_t* sample, int32_t* worker, int64_t* atoms_out, int64_t* split,
              int64_t* chunk_rank, int64_t* worker_atoms, int64_t* n_batches, int64_t* dropped);
/* Cost-model balancing (north_star "predicted atom/edge cost"; the reference
 * balances on atoms only, S/scheduler.cpp:62-158, and keeps a cost model only in
 * its simulator, H/simulator.hpp:22-27). Predicted per-sample cost
 *   cost = (per_sample + per_atom * atoms) + per_edge * edges
 * (edges: the sample's directed pair count, e.g. from lamm_neighbor_list_copy). */
typedef struct {
    double per_sample;
    double per_atom;
    double per_edge;
} lamm_cost_model;
/* cost[n] of each sample (edges nullable when per_edge == 0); LAMM_EINPUT on a
 * non-positive or non-finite cost. */
int lamm_sample_cost(const int64_t* atoms, const int64_t* edges, int64_t n, const lamm_cost_model* model,
                     double* cost);
/* lamm_plan with the balancing key = the predicted cost instead of the atom count:
 * the same shuffle, splits sorted by key, transpose chunk stream and greedy
 * least-loaded assignment (S/scheduler.cpp:91-158). With {0, 1, 0} it is
 * lamm_plan bit for bit. worker_cost [n_batches][workers] (nullable): predicted
 * per-worker cost of every mini-batch; the other outputs as lamm_plan. */
int lamm_plan_cost(const int64_t* atoms, const int64_t* edges, int64_t n, const lamm_cost_model* model,
                   int32_t workers, int32_t batch_per_worker, int32_t num_splits, uint64_t seed, int32_t mode,
                   int64_t* sample, int32_t* worker, int64_t* atoms_out, int64_t* split, int64_t* chunk_rank,
                   int64_t* worker_atoms, double* worker_cost, int64_t* n_batches, int64_t* dropped);
/* lamm::scheduler::schedule_metrics (S/scheduler.cpp:205-251). */
int lamm_schedule_metrics(int64_t n_batches, int32_t workers, int32_t batch_per_worker, const int32_t* worker,
                          const int64_t* atoms, const int64_t* split, const int64_t* chunk_rank,
                          double* max_imbalance, double* mean_imbalance, int64_t* monotonicity_violations,
                          int64_t* growth_events);

/* ------------------------------------------------- host: data layer --- */
/* The orchestration's data layer (S/trainer.cpp:64-125), host C++ in this library:
 * dataset::filter_max_atoms (S/dataset.cpp:85-96): indices of the samples with at
 * most `limit` atoms, in order. */
int lamm_filter_max_atoms(const int64_t* atom_ptr, int64_t n_samples, int64_t limit, int64_t* kept,
                          int64_t* n_kept);
/* dataset::split_train_val (S/dataset.cpp:98-111): Rng(seed).permutation(n), the
 * first llround(val_fraction * n) ids are validation; both sorted. */
int lamm_split_train_val(int64_t n, double val_fraction, uint64_t seed, int64_t* train, int64_t* n_train,
                         int64_t* val, int64_t* n_val);
/* denoise::apply_noise (S/denoise.cpp:7-40) of one system: noisy positions and
 * pseudo-force labels (either output nullable); scheme 1 centered, 0 baseline. */
int lamm_apply_noise(const double* positions, int64_t n_atoms, double sigma, int32_t scheme, uint64_t seed,
                     double* noisy, double* pseudo_forces);
/* estimate_pseudo_force_std (S/trainer.cpp:82-100): std of the pseudo-forces of the
 * first min(n_ids, 256) samples ids[v] (NULL: v) under seeds mix_seed(seed,
 * 0x50535444 + v). */
int lamm_pseudo_force_std(const int64_t* atom_ptr, const double* positions, const int64_t* ids, int64_t n_ids,
                          double sigma, int32_t scheme, uint64_t seed, double* out);
/* loss::DatasetNormalizer (H/loss.hpp:32-38): rho indexed by Z. */
typedef struct {
    double rho[119];
    uint8_t rho_has[119];
    double energy_mean;
    double energy_std;
    double force_std;
    uint8_t has_energy_stats;
} lamm_normalizer;
/* loss::fit_normalizer (S/loss.cpp:64-111) over the view's samples (masks and
 * labels as in lamm_batch_view; positions unused): per-element reference energies
 * by a minimum-norm least-squares solve (fit_reference, S/loss.cpp:17-48; complete
 * orthogonal decomposition, host_data.cpp), residual mean/std, force std (else
 * pseudo_force_std when > 0). */
int lamm_fit_normalizer(const lamm_batch_view* samples, double pseudo_force_std, lamm_normalizer* out);
/* model::reset_heads / init_heads (S/model.cpp:167-202): fresh energy head [H][heads]
 * and force head [2H+K][heads] from Rng(seed), bit-exact. */
int lamm_init_heads(const lamm_model_config* cfg, int32_t heads, uint64_t seed, double* energy_head,
                    double* force_head);

/* simulator::CostModel (H/simulator.hpp:22-27) and SimResult totals. */
typedef struct {
    double alpha_s;          /* per-worker fixed compute */
    double beta_s_per_atom;  /* compute per atom */
    double gamma_s;          /* allreduce constant */
    double delta_s;          /* penalty per high-water growth event */
} lamm_sim_cost;
typedef struct {
    double total_s;
    double throughput_samples_per_s;
    int64_t realloc_events;
    int64_t samples;
} lamm_sim_totals;
/* simulator::simulate (S/simulator.cpp:19-59) over a schedule's worker_atoms
 * [n_batches][workers] (lamm_plan output): per-step time, idle, realloc events and
 * max worker atoms (each output nullable), per-worker idle, totals; bit-exact with
 * the reference. worker_cost (nullable, extension): per-worker predicted seconds
 * [n_batches][workers] used in place of alpha + beta * atoms. */
int lamm_simulate(const int64_t* worker_atoms, const double* worker_cost, int64_t n_batches, int32_t workers,
                  int64_t samples_per_batch, const lamm_sim_cost* cost, double* step_time, double* step_idle,
                  int32_t* step_realloc, int64_t* step_max_atoms, double* worker_idle, lamm_sim_totals* totals);

/* ----------------------------------------------- host: data generation --- */
/* lamm::trace::make_trace (S/trace.cpp:50-76). kind: 0 constant, 1 uniform,
 * 2 lognormal, 3 bimodal. */
int lamm_make_trace(int32_t kind, int64_t count, int64_t min_atoms, int64_t max_atoms, double constant_atoms,
                    double mode, double sigma, double mode_a, double sigma_a, double mode_b, double sigma_b,
                    double weight_a, uint64_t seed, int64_t* out);
/* lamm::dataset::temperature_counts / build_epoch_index (S/dataset.cpp:39-83). */
int lamm_temperature_counts(const double* sizes, int32_t k, double temperature, double* out);
int lamm_build_epoch_index(const double* repeats, const int64_t* sizes, int32_t k, uint64_t seed, int64_t cap,
                           int32_t* out_subset, int64_t* out_sample, int64_t* count);
/* lamm::dataset::synth_generate (S/dataset.cpp:234-247) with the default
 * Morse table: first the per-sample atom counts (atom_ptr[count+1]), then the
 * packed samples. task: 0 energy_and_forces, 1 energy_only, 2 denoising. */
int lamm_synth_counts(int64_t count, double mode, double sigma, int32_t min_atoms, int32_t max_atoms,
                      uint64_t seed, int64_t* atom_ptr);
int lamm_synth_fill(int32_t task, int64_t count, double mode, double sigma, int32_t min_atoms, int32_t max_atoms,
                    const int32_t* elements, int32_t n_elements, int32_t relax_steps, double relax_step,
                    double energy_scale, const int32_t* offset_z, const double* offset_value, int32_t n_offsets,
                    uint64_t seed, int32_t threads, const int64_t* atom_ptr, double* positions,
                    int32_t* atomic_numbers, uint8_t* energy_mask, uint8_t* force_mask, double* energy,
                    double* forces);
/* ------------------------------------------------------ on-disk formats --- */
/* LAMMCKPT checkpoints, byte-compatible with lamm::model::save_checkpoint /
 * load_checkpoint (H/model.hpp:131-139, S/model.cpp:429-497): params flat in
 * for_each_tensor order. load with params == NULL returns the config and the
 * parameter count only. */
int lamm_checkpoint_save(const char* path, const lamm_model_config* cfg, const double* params, size_t n);
int lamm_checkpoint_load(const char* path, lamm_model_config* cfg, double* params, size_t cap, size_t* n_out);
/* The RMS optimizer state v in the same layout (magic "LAMMRMS1"; the reference
 * keeps it in memory only), for bit-exact resumption. */
int lamm_rms_state_save(const char* path, const lamm_model_config* cfg, const double* v, size_t n);
int lamm_rms_state_load(const char* path, lamm_model_config* cfg, double* v, size_t cap, size_t* n_out);
/* LAMMDS1 catalog subsets (S/dataset.cpp:273-330) read straight into the packed
 * batch layout of lamm_batch_view: info gives the sample and atom counts to size
 * the arrays (atom_ptr[count+1], positions[3N], Z[N], per-sample masks/energy,
 * forces[3N]); dataset_index is set to head_index (read_catalog). info reads
 * through the records (a truncated file is LAMM_EINPUT); read refuses files with
 * more than sample_cap samples or atom_cap atoms (the sizes of the arrays). */
int lamm_subset_info(const char* path, int64_t* count, int64_t* total_atoms);
int lamm_subset_read(const char* path, int32_t head_index, int64_t sample_cap, int64_t atom_cap,
                     int64_t* atom_ptr, double* positions, int32_t* atomic_numbers, int32_t* dataset_index,
                     uint8_t* energy_mask, uint8_t* force_mask, double* energy, double* forces);

/* Inverse of a 3x3 cell (row-major, rows = lattice vectors) by cofactors: the
 * exact bits the minimum-image test uses. Returns LAMM_EINPUT if singular. */
int lamm_cell_inverse(const double* cell, double* out);

/* Reference RNG streams (H/rng.hpp): mix_seed and Box-Muller normals. */
uint64_t lamm_mix_seed(uint64_t a, uint64_t b);
int lamm_rng_normals(uint64_t seed, int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif /* LAMM_B200_H */
