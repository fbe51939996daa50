// oracle/ref_capi.cpp - C-ABI shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. This file is compiled together with the reference's
// own sources, straight from /root/reference/proj/core/src/*.cpp (never copied
// into this repo), into oracle/_ref/liblamm_ref.so by oracle/Makefile. Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs load it, and only as the checker or the CPU baseline.
//
// Every entry point forwards to the reference's public C++ API; the one
// exception is the RMS optimizer, which the reference keeps file-local
// (S/trainer.cpp:29-54) and which is restated here line for line so the
// train-step replica (S/trainer.cpp:258-327) can run outside run_loop.
//
// Packed-batch conventions shared with oracle/lamm_oracle.c and the product:
//   atom_ptr[B+1] (int64), positions[3N] (f64, atom-major xyz), Z[N] (int32),
//   dataset_index[B], energy_mask[B], force_mask[B], energy[B], forces[3N],
//   denoise[B] (1: sample is drawn from a denoising subset).
//   Predictions: energy[B*D]; forces: per-sample block at 3*D*atom_ptr[s],
//   inside it the reference layout (d*n + j)*3 + c (H/model.hpp:99-108).
//   Parameters: flat, for_each_tensor order (H/model.hpp:59-66), row-major.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "lamm/core.hpp"
#include "lamm/dataset.hpp"
#include "lamm/denoise.hpp"
#include "lamm/loss.hpp"
#include "lamm/model.hpp"
#include "lamm/rng.hpp"
#include "lamm/scheduler.hpp"
#include "lamm/simulator.hpp"
#include "lamm/trace.hpp"
#include "lamm/trainer.hpp"

#define LREF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const lamm::InputError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

lamm::model::ModelConfig make_cfg(int H, int L, int K, double rc, int D) {
    lamm::model::ModelConfig c;
    c.hidden = H;
    c.layers = L;
    c.rbf = K;
    c.cutoff = rc;
    c.heads = D;
    return c;
}

lamm::model::ModelParams params_from_flat(const lamm::model::ModelConfig& cfg, const double* flat) {
    auto p = lamm::model::init_params(cfg, 0);
    std::size_t off = 0;
    lamm::model::for_each_tensor(p, [&](lamm::Matrix& m) {
        std::memcpy(m.data(), flat + off, m.size() * sizeof(double));
        off += m.size();
    });
    return p;
}

void params_to_flat(const lamm::model::ModelParams& p, double* flat) {
    std::size_t off = 0;
    lamm::model::for_each_tensor(p, [&](const lamm::Matrix& m) {
        std::memcpy(flat + off, m.data(), m.size() * sizeof(double));
        off += m.size();
    });
}

lamm::AtomicSystem system_at(const int64_t* atom_ptr, const double* pos, const int32_t* Z, int s) {
    lamm::AtomicSystem sys;
    for (int64_t a = atom_ptr[s]; a < atom_ptr[s + 1]; ++a) {
        sys.positions.push_back({pos[3 * a], pos[3 * a + 1], pos[3 * a + 2]});
        sys.atomic_numbers.push_back(Z[a]);
    }
    return sys;
}

lamm::Sample sample_at(const int64_t* atom_ptr, const double* pos, const int32_t* Z, const int32_t* dsidx,
                       const uint8_t* emask, const uint8_t* fmask, const double* energy, const double* forces,
                       int s) {
    lamm::Sample out;
    out.system = system_at(atom_ptr, pos, Z, s);
    out.labels.dataset_index = dsidx ? dsidx[s] : 0;
    out.labels.energy_mask = emask && emask[s];
    out.labels.force_mask = fmask && fmask[s];
    if (out.labels.energy_mask) out.labels.energy = energy[s];
    if (out.labels.force_mask)
        for (int64_t a = atom_ptr[s]; a < atom_ptr[s + 1]; ++a)
            out.labels.forces.push_back({forces[3 * a], forces[3 * a + 1], forces[3 * a + 2]});
    out.subset_id = out.labels.dataset_index;
    return out;
}

lamm::loss::ReferenceTable table_from(int ntab, const double* rho, const uint8_t* rho_has, const double* mean,
                                      const double* stdv, const double* fstd, const uint8_t* has) {
    lamm::loss::ReferenceTable t;
    t.per_dataset.resize(static_cast<std::size_t>(ntab));
    for (int d = 0; d < ntab; ++d) {
        auto& n = t.per_dataset[static_cast<std::size_t>(d)];
        for (int z = 1; z <= 118; ++z)
            if (rho_has[d * 119 + z]) n.reference_energies[z] = rho[d * 119 + z];
        n.energy_mean = mean[d];
        n.energy_std = stdv[d];
        n.force_std = fstd[d];
        n.has_energy_stats = has[d] != 0;
    }
    return t;
}

// S/trainer.cpp:17-26 stream tags used by the step body.
constexpr std::uint64_t kNoiseTag = 0x4e4f4953;

}  // namespace

LREF_API const char* lref_last_error() { return g_err.c_str(); }

LREF_API uint64_t lref_mix_seed(uint64_t a, uint64_t b) { return lamm::mix_seed(a, b); }

LREF_API void lref_rng_normals(uint64_t seed, int64_t n, double* out) {
    lamm::Rng r(seed);
    for (int64_t k = 0; k < n; ++k) out[k] = r.normal();
}

LREF_API void lref_rng_uniforms(uint64_t seed, int64_t n, double* out) {
    lamm::Rng r(seed);
    for (int64_t k = 0; k < n; ++k) out[k] = r.uniform();
}

LREF_API void lref_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
    lamm::Rng r(seed);
    for (int64_t k = 0; k < n; ++k) out[k] = r.next_u64();
}

LREF_API void lref_rng_bounded(uint64_t seed, int64_t n, uint64_t bound, uint64_t* out) {
    lamm::Rng r(seed);
    for (int64_t k = 0; k < n; ++k) out[k] = r.bounded(bound);
}

LREF_API void lref_rng_permutation(uint64_t seed, int64_t n, int64_t* out) {
    lamm::Rng r(seed);
    const auto p = r.permutation(static_cast<std::size_t>(n));
    for (int64_t k = 0; k < n; ++k) out[k] = static_cast<int64_t>(p[static_cast<std::size_t>(k)]);
}

// ---- geometry (S/core.cpp:30-48) -----------------------------------------
LREF_API int64_t lref_neighbor_list(int32_t n, const double* pos, const int32_t* Z, double cutoff, int64_t cap,
                                    int32_t* oi, int32_t* oj, double* odist, double* ounit) {
    int64_t count = -1;
    const int st = guarded([&] {
        const int64_t ptr[2] = {0, n};
        const auto nl = lamm::build_neighbor_list(system_at(ptr, pos, Z, 0), cutoff);
        count = static_cast<int64_t>(nl.pairs.size());
        for (int64_t p = 0; p < std::min(count, cap); ++p) {
            const auto& q = nl.pairs[static_cast<std::size_t>(p)];
            oi[p] = q.i;
            oj[p] = q.j;
            odist[p] = q.distance;
            for (int c = 0; c < 3; ++c) ounit[3 * p + c] = q.unit[static_cast<std::size_t>(c)];
        }
    });
    return st == 0 ? count : -static_cast<int64_t>(st);
}

// ---- model (S/model.cpp) ------------------------------------------------------
LREF_API int64_t lref_param_count(int H, int L, int K, int D) {
    return 118LL * H + (int64_t)L * H * K + (int64_t)L * H * H + (int64_t)H * D + (int64_t)(2 * H + K) * D;
}

LREF_API int lref_init_params(int H, int L, int K, double rc, int D, uint64_t seed, double* out) {
    return guarded([&] { params_to_flat(lamm::model::init_params(make_cfg(H, L, K, rc, D), seed), out); });
}

LREF_API int lref_forward(int H, int L, int K, double rc, int D, const double* params, int32_t B,
                          const int64_t* atom_ptr, const double* pos, const int32_t* Z, double* out_energy,
                          double* out_forces) {
    return guarded([&] {
        const auto cfg = make_cfg(H, L, K, rc, D);
        const auto p = params_from_flat(cfg, params);
        for (int s = 0; s < B; ++s) {
            const auto pred = lamm::model::forward(system_at(atom_ptr, pos, Z, s), p, cfg, nullptr);
            std::memcpy(out_energy + (int64_t)s * D, pred.energy.data(), sizeof(double) * D);
            std::memcpy(out_forces + 3 * D * atom_ptr[s], pred.forces.data(), sizeof(double) * pred.forces.size());
        }
    });
}

/// One sample's ForwardCache (H/model.hpp:86-95): h[0..L] and tanh(m)[0..L-1].
LREF_API int lref_forward_cache(int H, int L, int K, double rc, int D, const double* params, int32_t n,
                                const double* pos, const int32_t* Z, double* h_all, double* mt_all) {
    return guarded([&] {
        const auto cfg = make_cfg(H, L, K, rc, D);
        const auto p = params_from_flat(cfg, params);
        const int64_t ptr[2] = {0, n};
        lamm::model::ForwardCache cache;
        lamm::model::forward(system_at(ptr, pos, Z, 0), p, cfg, &cache);
        for (int l = 0; l <= L; ++l)
            std::memcpy(h_all + (int64_t)l * n * H, cache.h[static_cast<std::size_t>(l)].data(),
                        sizeof(double) * n * H);
        for (int l = 0; l < L; ++l)
            std::memcpy(mt_all + (int64_t)l * n * H, cache.msg_tanh[static_cast<std::size_t>(l)].data(),
                        sizeof(double) * n * H);
    });
}

LREF_API int lref_backward(int H, int L, int K, double rc, int D, const double* params, int32_t B,
                           const int64_t* atom_ptr, const double* pos, const int32_t* Z, const double* up_energy,
                           const double* up_forces, double* grads_accum) {
    return guarded([&] {
        const auto cfg = make_cfg(H, L, K, rc, D);
        const auto p = params_from_flat(cfg, params);
        auto g = params_from_flat(cfg, grads_accum);
        for (int s = 0; s < B; ++s) {
            lamm::model::ForwardCache cache;
            const auto sys = system_at(atom_ptr, pos, Z, s);
            lamm::model::forward(sys, p, cfg, &cache);
            lamm::model::PredictionGrad up;
            up.n_atoms = static_cast<int>(sys.size());
            up.heads = D;
            up.energy.assign(up_energy + (int64_t)s * D, up_energy + (int64_t)(s + 1) * D);
            up.forces.assign(up_forces + 3 * D * atom_ptr[s], up_forces + 3 * D * atom_ptr[s + 1]);
            lamm::model::backward(cache, p, cfg, up, g);
        }
        params_to_flat(g, grads_accum);
    });
}

// ---- evaluation (S/trainer.cpp:491-553) -------------------------------------
/// trainer::evaluate on a packed batch with raw labels; out = {energy_mae,
/// force_mae, energy_count, force_count} (MAEs in meV, NaN without labels).
LREF_API int lref_evaluate(int H, int L, int K, double rc, int D, const double* params, int32_t B,
                           const int64_t* atom_ptr, const double* pos, const int32_t* Z, const int32_t* dsidx,
                           const uint8_t* emask, const uint8_t* fmask, const double* energy, const double* forces,
                           int ntab, const double* rho, const uint8_t* rho_has, const double* mean,
                           const double* stdv, const double* fstd, const uint8_t* has, double* out) {
    return guarded([&] {
        const auto cfg = make_cfg(H, L, K, rc, D);
        const auto p = params_from_flat(cfg, params);
        const auto t = table_from(ntab, rho, rho_has, mean, stdv, fstd, has);
        std::vector<lamm::Sample> samples;
        for (int s = 0; s < B; ++s)
            samples.push_back(sample_at(atom_ptr, pos, Z, dsidx, emask, fmask, energy, forces, s));
        const auto r = lamm::trainer::evaluate(cfg, p, t, samples);
        out[0] = r.energy_mae;
        out[1] = r.force_mae;
        out[2] = static_cast<double>(r.energy_count);
        out[3] = static_cast<double>(r.force_count);
    });
}

// ---- loss (S/loss.cpp) ------------------------------------------------------
LREF_API int lref_normalize_labels(int32_t B, const int64_t* atom_ptr, const double* pos, const int32_t* Z,
                                   const int32_t* dsidx, const uint8_t* emask, const uint8_t* fmask,
                                   const double* energy, const double* forces, int ntab, const double* rho,
                                   const uint8_t* rho_has, const double* mean, const double* stdv,
                                   const double* fstd, const uint8_t* has, double* out_energy, double* out_forces) {
    return guarded([&] {
        const auto t = table_from(ntab, rho, rho_has, mean, stdv, fstd, has);
        for (int s = 0; s < B; ++s) {
            const auto in = sample_at(atom_ptr, pos, Z, dsidx, emask, fmask, energy, forces, s);
            const auto o = lamm::loss::normalize_labels(in, t);
            out_energy[s] = o.labels.energy_mask ? *o.labels.energy : 0.0;
            for (int64_t a = atom_ptr[s]; a < atom_ptr[s + 1]; ++a)
                for (int c = 0; c < 3; ++c)
                    out_forces[3 * a + c] =
                        o.labels.force_mask ? o.labels.forces[static_cast<std::size_t>(a - atom_ptr[s])][c] : 0.0;
        }
    });
}

/// masked_loss_grad (S/loss.cpp:222-226). breakdown = {total, energy_term,
/// force_term, energy_labeled, force_labeled, energy_empty, force_empty}.
LREF_API int lref_loss_grad(int32_t B, const int64_t* atom_ptr, int D, const int32_t* dsidx, const uint8_t* emask,
                            const uint8_t* fmask, const double* energy, const double* forces,
                            const double* pred_energy, const double* pred_forces, double lambda_e, double lambda_f,
                            double* breakdown, double* g_energy, double* g_forces) {
    return guarded([&] {
        std::vector<lamm::Sample> batch;
        std::vector<lamm::model::Prediction> preds;
        for (int s = 0; s < B; ++s) {
            // positions are irrelevant to the loss; zeros keep the shapes valid
            lamm::Sample smp;
            const int64_t n = atom_ptr[s + 1] - atom_ptr[s];
            smp.system.positions.assign(static_cast<std::size_t>(n), {0.0, 0.0, 0.0});
            smp.system.atomic_numbers.assign(static_cast<std::size_t>(n), 1);
            smp.labels.dataset_index = dsidx[s];
            smp.labels.energy_mask = emask[s];
            smp.labels.force_mask = fmask[s];
            if (emask[s]) smp.labels.energy = energy[s];
            if (fmask[s])
                for (int64_t a = atom_ptr[s]; a < atom_ptr[s + 1]; ++a)
                    smp.labels.forces.push_back({forces[3 * a], forces[3 * a + 1], forces[3 * a + 2]});
            batch.push_back(std::move(smp));
            lamm::model::Prediction p;
            p.n_atoms = static_cast<int>(n);
            p.heads = D;
            p.energy.assign(pred_energy + (int64_t)s * D, pred_energy + (int64_t)(s + 1) * D);
            p.forces.assign(pred_forces + 3 * D * atom_ptr[s], pred_forces + 3 * D * atom_ptr[s + 1]);
            preds.push_back(std::move(p));
        }
        std::vector<lamm::model::PredictionGrad> g;
        const lamm::loss::LossConfig lc{lambda_e, lambda_f};
        const auto b = lamm::loss::masked_loss_grad(batch, preds, lc, g);
        breakdown[0] = b.total;
        breakdown[1] = b.energy_term;
        breakdown[2] = b.force_term;
        breakdown[3] = b.energy_labeled;
        breakdown[4] = b.force_labeled;
        breakdown[5] = b.energy_empty;
        breakdown[6] = b.force_empty;
        for (int s = 0; s < B; ++s) {
            std::memcpy(g_energy + (int64_t)s * D, g[static_cast<std::size_t>(s)].energy.data(), sizeof(double) * D);
            std::memcpy(g_forces + 3 * D * atom_ptr[s], g[static_cast<std::size_t>(s)].forces.data(),
                        sizeof(double) * g[static_cast<std::size_t>(s)].forces.size());
        }
    });
}

// ---- denoise (S/denoise.cpp) ------------------------------------------------
LREF_API int lref_apply_noise(int32_t n, const double* pos, const int32_t* Z, double sigma, int scheme,
                              uint64_t seed, double* noisy, double* labels) {
    return guarded([&] {
        const int64_t ptr[2] = {0, n};
        lamm::denoise::NoiseConfig c;
        c.sigma = sigma;
        c.scheme = scheme ? lamm::denoise::Scheme::centered : lamm::denoise::Scheme::baseline;
        c.seed = seed;
        const auto r = lamm::denoise::apply_noise(system_at(ptr, pos, Z, 0), c);
        for (int a = 0; a < n; ++a)
            for (int k = 0; k < 3; ++k) {
                noisy[3 * a + k] = r.noisy.positions[static_cast<std::size_t>(a)][k];
                labels[3 * a + k] = r.pseudo_forces[static_cast<std::size_t>(a)][k];
            }
    });
}

LREF_API int lref_apply_displacements(int32_t n, const double* pos, const int32_t* Z, const double* deltas,
                                      int scheme, double* noisy, double* labels) {
    return guarded([&] {
        const int64_t ptr[2] = {0, n};
        std::vector<lamm::Vec3> d(static_cast<std::size_t>(n));
        for (int a = 0; a < n; ++a) d[static_cast<std::size_t>(a)] = {deltas[3 * a], deltas[3 * a + 1], deltas[3 * a + 2]};
        const auto r = lamm::denoise::apply_displacements(
            system_at(ptr, pos, Z, 0), d, scheme ? lamm::denoise::Scheme::centered : lamm::denoise::Scheme::baseline);
        for (int a = 0; a < n; ++a)
            for (int k = 0; k < 3; ++k) {
                noisy[3 * a + k] = r.noisy.positions[static_cast<std::size_t>(a)][k];
                labels[3 * a + k] = r.pseudo_forces[static_cast<std::size_t>(a)][k];
            }
    });
}

// ---- train-step replica (S/trainer.cpp:258-327) ----------------------------
/// One optimizer step over G*B packed samples in worker-major order (the order
/// pack_batch guarantees, S/scheduler.cpp:43-58). params and v (RMS state) are
/// updated in place. out_grads (nullable) receives the worker-averaged,
/// pre-clip gradient. threads > 1 runs each worker's forward/backward over
/// samples in parallel with per-thread gradient buffers summed in a fixed
/// order (deterministic, but not bit-identical to threads == 1).
/// Returns 5 on a non-finite loss or gradient (S/trainer.cpp:322-324).
LREF_API int lref_train_step(int H, int L, int K, double rc, int D, int G, int B, const int64_t* atom_ptr,
                             const double* pos, const int32_t* Z, const int32_t* dsidx, const uint8_t* emask,
                             const uint8_t* fmask, const double* energy, const double* forces,
                             const uint8_t* denoise_flag, int ntab, const double* rho, const uint8_t* rho_has,
                             const double* mean, const double* stdv, const double* fstd, const uint8_t* has,
                             double noise_sigma, int noise_scheme, uint64_t seed, int64_t step, double lambda_e,
                             double lambda_f, double lr, double clip, double decay, double eps, double* params,
                             double* rms_v, double* out_loss, double* out_grad_norm, double* out_grads, int threads) {
    int status = 0;
    const int st = guarded([&] {
        const auto cfg = make_cfg(H, L, K, rc, D);
        auto p = params_from_flat(cfg, params);
        auto v = params_from_flat(cfg, rms_v);
        const auto refs = table_from(ntab, rho, rho_has, mean, stdv, fstd, has);
        const lamm::loss::LossConfig lcfg{lambda_e, lambda_f};
        double loss_sum = 0.0;
        auto grads = lamm::model::zero_like(p);
        for (int g = 0; g < G; ++g) {
            std::vector<lamm::Sample> normalized(static_cast<std::size_t>(B));
            std::vector<lamm::model::ForwardCache> caches(static_cast<std::size_t>(B));
            std::vector<lamm::model::Prediction> preds(static_cast<std::size_t>(B));
            auto prep = [&](int b) {
                const int pos_ = g * B + b;
                lamm::Sample raw;
                if (denoise_flag && denoise_flag[pos_]) {
                    lamm::denoise::NoiseConfig ncfg{
                        noise_sigma,
                        noise_scheme ? lamm::denoise::Scheme::centered : lamm::denoise::Scheme::baseline,
                        lamm::mix_seed(lamm::mix_seed(seed, kNoiseTag + static_cast<std::uint64_t>(step)),
                                       static_cast<std::uint64_t>(pos_))};
                    raw = lamm::denoise::make_denoising_sample(system_at(atom_ptr, pos, Z, pos_), ncfg, dsidx[pos_],
                                                               dsidx[pos_]);
                } else {
                    raw = sample_at(atom_ptr, pos, Z, dsidx, emask, fmask, energy, forces, pos_);
                }
                normalized[static_cast<std::size_t>(b)] = lamm::loss::normalize_labels(raw, refs);
                preds[static_cast<std::size_t>(b)] = lamm::model::forward(
                    normalized[static_cast<std::size_t>(b)].system, p, cfg, &caches[static_cast<std::size_t>(b)]);
            };
            const int nt = std::max(1, std::min(threads, B));
            if (nt <= 1) {
                for (int b = 0; b < B; ++b) prep(b);
            } else {
                std::vector<std::thread> pool;
                for (int t = 0; t < nt; ++t)
                    pool.emplace_back([&, t] {
                        for (int b = t; b < B; b += nt) prep(b);
                    });
                for (auto& th : pool) th.join();
            }
            std::vector<lamm::model::PredictionGrad> pgrads;
            const auto breakdown = lamm::loss::masked_loss_grad(normalized, preds, lcfg, pgrads);
            loss_sum += breakdown.total;
            if (nt <= 1) {
                for (int b = 0; b < B; ++b)
                    lamm::model::backward(caches[static_cast<std::size_t>(b)], p, cfg,
                                          pgrads[static_cast<std::size_t>(b)], grads);
            } else {
                std::vector<lamm::model::Gradients> part(static_cast<std::size_t>(nt), lamm::model::zero_like(p));
                std::vector<std::thread> pool;
                for (int t = 0; t < nt; ++t)
                    pool.emplace_back([&, t] {
                        for (int b = t; b < B; b += nt)
                            lamm::model::backward(caches[static_cast<std::size_t>(b)], p, cfg,
                                                  pgrads[static_cast<std::size_t>(b)], part[static_cast<std::size_t>(t)]);
                    });
                for (auto& th : pool) th.join();
                for (int t = 0; t < nt; ++t) lamm::model::axpy_params(grads, part[static_cast<std::size_t>(t)], 1.0);
            }
        }
        lamm::model::scale_params(grads, 1.0 / static_cast<double>(G));
        const double loss = loss_sum / static_cast<double>(G);
        const double grad_norm = lamm::model::global_norm(grads);
        *out_loss = loss;
        *out_grad_norm = grad_norm;
        if (out_grads) params_to_flat(grads, out_grads);
        if (!std::isfinite(loss) || !std::isfinite(grad_norm)) {
            status = 5;
            g_err = "non-finite loss or gradient at step " + std::to_string(step);
            return;
        }
        if (clip > 0.0 && grad_norm > clip) lamm::model::scale_params(grads, clip / grad_norm);
        // RmsOptimizer::step, S/trainer.cpp:37-53 (file-local in the reference)
        std::vector<const lamm::Matrix*> gl;
        lamm::model::for_each_tensor(grads, [&](const lamm::Matrix& m) { gl.push_back(&m); });
        std::vector<lamm::Matrix*> vl;
        lamm::model::for_each_tensor(v, [&](lamm::Matrix& m) { vl.push_back(&m); });
        std::size_t t = 0;
        lamm::model::for_each_tensor(p, [&](lamm::Matrix& pm) {
            const lamm::Matrix& gm = *gl.at(t);
            lamm::Matrix& vm = *vl.at(t);
            ++t;
            for (std::size_t k = 0; k < pm.size(); ++k) {
                const double gk = gm.data()[k];
                vm.data()[k] = decay * vm.data()[k] + (1.0 - decay) * gk * gk;
                pm.data()[k] -= lr * gk / (std::sqrt(vm.data()[k]) + eps);
            }
        });
        params_to_flat(p, params);
        params_to_flat(v, rms_v);
    });
    return st != 0 ? st : status;
}

// ---- scheduler (S/scheduler.cpp) ---------------------------------------------
namespace {
struct PlanHandle {
    lamm::scheduler::MiniBatchSchedule s;
};
}  // namespace

LREF_API void* lref_plan(const int64_t* atoms, int64_t n, int G, int B, int S, uint64_t seed, int mode) {
    PlanHandle* h = nullptr;
    const int st = guarded([&] {
        lamm::scheduler::ScheduleConfig c;
        c.workers = G;
        c.batch_per_worker = B;
        c.num_splits = S;
        c.seed = seed;
        c.mode = mode == 0 ? lamm::scheduler::Mode::balanced
                           : (mode == 1 ? lamm::scheduler::Mode::greedy_only : lamm::scheduler::Mode::naive);
        auto hp = std::make_unique<PlanHandle>();
        hp->s = lamm::scheduler::plan(std::vector<int64_t>(atoms, atoms + n), c);
        h = hp.release();
    });
    return st == 0 ? h : nullptr;
}

LREF_API void lref_plan_info(void* h, int64_t* nbatches, int64_t* dropped) {
    auto* p = static_cast<PlanHandle*>(h);
    *nbatches = static_cast<int64_t>(p->s.batches.size());
    *dropped = p->s.dropped_samples;
}

/// Flat (step-major, then in-batch order) copies of every ScheduledSample.
LREF_API void lref_plan_copy(void* h, int64_t* sample, int32_t* worker, int64_t* atoms, int64_t* split,
                             int64_t* chunk_rank, int64_t* worker_atoms) {
    auto* p = static_cast<PlanHandle*>(h);
    int64_t k = 0, w = 0;
    for (const auto& b : p->s.batches) {
        for (const auto& s : b.samples) {
            sample[k] = s.sample;
            worker[k] = s.worker;
            atoms[k] = s.atoms;
            split[k] = s.split;
            chunk_rank[k] = s.chunk_rank;
            ++k;
        }
        for (auto a : b.worker_atoms) worker_atoms[w++] = a;
    }
}

LREF_API void lref_schedule_metrics(void* h, double* max_imb, double* mean_imb, int64_t* mono, int64_t* growth) {
    const auto m = lamm::scheduler::schedule_metrics(static_cast<PlanHandle*>(h)->s);
    *max_imb = m.max_imbalance;
    *mean_imb = m.mean_imbalance;
    *mono = m.monotonicity_violations;
    *growth = static_cast<int64_t>(m.growth_events.size());
}

LREF_API void lref_plan_free(void* h) { delete static_cast<PlanHandle*>(h); }

LREF_API int lref_greedy_assign(const int64_t* atoms, int64_t n, int G, int B, int32_t* out) {
    return guarded([&] {
        const auto a = lamm::scheduler::greedy_assign(std::vector<int64_t>(atoms, atoms + n), G, B);
        for (int64_t k = 0; k < n; ++k) out[k] = a[static_cast<std::size_t>(k)];
    });
}

// ---- trace / dataset (S/trace.cpp, S/dataset.cpp) ----------------------------
LREF_API int lref_make_trace(int kind, int64_t count, int64_t min_atoms, int64_t max_atoms, double constant_atoms,
                             double mode, double sigma, double mode_a, double sigma_a, double mode_b, double sigma_b,
                             double weight_a, uint64_t seed, int64_t* out) {
    return guarded([&] {
        lamm::trace::TraceSpec s;
        s.kind = static_cast<lamm::trace::Kind>(kind);
        s.count = count;
        s.min_atoms = min_atoms;
        s.max_atoms = max_atoms;
        s.constant_atoms = constant_atoms;
        s.mode = mode;
        s.sigma = sigma;
        s.mode_a = mode_a;
        s.sigma_a = sigma_a;
        s.mode_b = mode_b;
        s.sigma_b = sigma_b;
        s.weight_a = weight_a;
        const auto t = lamm::trace::make_trace(s, seed);
        std::memcpy(out, t.data(), sizeof(int64_t) * t.size());
    });
}

LREF_API int lref_temperature_counts(const double* sizes, int k, double T, double* out) {
    return guarded([&] {
        const auto r = lamm::dataset::temperature_counts(std::vector<double>(sizes, sizes + k), T);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

LREF_API int64_t lref_build_epoch_index(const double* repeats, const int64_t* sizes, int k, uint64_t seed,
                                        int64_t cap, int32_t* out_subset, int64_t* out_sample) {
    int64_t count = -1;
    const int st = guarded([&] {
        lamm::dataset::MixPlan plan;
        plan.repeats.assign(repeats, repeats + k);
        const auto e = lamm::dataset::build_epoch_index(plan, std::vector<int64_t>(sizes, sizes + k), seed);
        count = static_cast<int64_t>(e.size());
        for (int64_t q = 0; q < std::min(count, cap); ++q) {
            out_subset[q] = e[static_cast<std::size_t>(q)].subset;
            out_sample[q] = e[static_cast<std::size_t>(q)].sample;
        }
    });
    return st == 0 ? count : -static_cast<int64_t>(st);
}

namespace {
struct SamplesHandle {
    std::vector<lamm::Sample> v;
};
}  // namespace

/// synth_generate (S/dataset.cpp:234-247) with the default Morse table and an
/// optional per-element label offset transform.
LREF_API void* lref_synth_generate(int task, int64_t count, double mode, double sigma, int min_atoms, int max_atoms,
                                   const int32_t* elements, int nelem, int relax_steps, double relax_step,
                                   double energy_scale, const int32_t* off_z, const double* off_v, int noff,
                                   uint64_t seed) {
    SamplesHandle* h = nullptr;
    guarded([&] {
        lamm::dataset::SynthSpec s;
        s.task = static_cast<lamm::dataset::TaskKind>(task);
        s.count = count;
        s.atom_count_mode = mode;
        s.atom_count_sigma = sigma;
        s.min_atoms = min_atoms;
        s.max_atoms = max_atoms;
        s.elements.assign(elements, elements + nelem);
        s.relax_steps = relax_steps;
        s.relax_step = relax_step;
        s.transform.energy_scale = energy_scale;
        for (int q = 0; q < noff; ++q) s.transform.element_offsets[off_z[q]] = off_v[q];
        auto hp = std::make_unique<SamplesHandle>();
        hp->v = lamm::dataset::synth_generate(s, count, seed);
        h = hp.release();
    });
    return h;
}

LREF_API void lref_samples_info(void* h, int64_t* count, int64_t* total_atoms) {
    auto* p = static_cast<SamplesHandle*>(h);
    *count = static_cast<int64_t>(p->v.size());
    int64_t t = 0;
    for (const auto& s : p->v) t += static_cast<int64_t>(s.system.size());
    *total_atoms = t;
}

LREF_API void lref_samples_copy(void* h, int64_t* atom_ptr, double* pos, int32_t* Z, uint8_t* emask, uint8_t* fmask,
                                double* energy, double* forces) {
    auto* p = static_cast<SamplesHandle*>(h);
    int64_t a = 0;
    atom_ptr[0] = 0;
    for (std::size_t s = 0; s < p->v.size(); ++s) {
        const auto& smp = p->v[s];
        emask[s] = smp.labels.energy_mask;
        fmask[s] = smp.labels.force_mask;
        energy[s] = smp.labels.energy.value_or(0.0);
        for (std::size_t k = 0; k < smp.system.size(); ++k, ++a) {
            for (int c = 0; c < 3; ++c) {
                pos[3 * a + c] = smp.system.positions[k][c];
                forces[3 * a + c] = smp.labels.force_mask ? smp.labels.forces[k][c] : 0.0;
            }
            Z[a] = smp.system.atomic_numbers[k];
        }
        atom_ptr[s + 1] = a;
    }
}

LREF_API void lref_samples_free(void* h) { delete static_cast<SamplesHandle*>(h); }

// ---- on-disk formats (S/dataset.cpp:273-393, S/model.cpp:429-497) -----------
/// synth_catalog of three small subsets (energy+forces, energy-only, denoising)
/// written with write_catalog into dir.
LREF_API int lref_write_demo_catalog(const char* dir, int64_t count, uint64_t seed) {
    return guarded([&] {
        std::vector<lamm::dataset::SynthSpec> specs(3);
        const char* names[3] = {"ef", "energy", "denoise"};
        for (int k = 0; k < 3; ++k) {
            specs[k].name = names[k];
            specs[k].task = static_cast<lamm::dataset::TaskKind>(k);
            specs[k].count = count;
            specs[k].atom_count_mode = 10.0 + 5.0 * k;
            specs[k].min_atoms = 2;
            specs[k].max_atoms = 40;
            specs[k].elements = {1, 6, 7, 8};
        }
        lamm::dataset::write_catalog(dir, lamm::dataset::synth_catalog(specs, seed));
    });
}

/// read_catalog: every subset's samples concatenated (dataset_index = head_index).
LREF_API void* lref_read_catalog(const char* dir, int32_t* n_subsets, int64_t* subset_sizes) {
    SamplesHandle* h = nullptr;
    guarded([&] {
        const auto cat = lamm::dataset::read_catalog(dir);
        auto hp = std::make_unique<SamplesHandle>();
        *n_subsets = static_cast<int32_t>(cat.subsets.size());
        for (std::size_t k = 0; k < cat.subsets.size(); ++k) {
            subset_sizes[k] = static_cast<int64_t>(cat.subsets[k].samples.size());
            for (const auto& smp : cat.subsets[k].samples) hp->v.push_back(smp);
        }
        h = hp.release();
    });
    return h;
}

LREF_API void lref_samples_heads(void* h, int32_t* dataset_index) {
    auto* p = static_cast<SamplesHandle*>(h);
    for (std::size_t s = 0; s < p->v.size(); ++s) dataset_index[s] = p->v[s].labels.dataset_index;
}

LREF_API int lref_checkpoint_save(const char* path, int H, int L, int K, double rc, int D, const double* params) {
    return guarded([&] {
        const auto cfg = make_cfg(H, L, K, rc, D);
        lamm::model::save_checkpoint(path, cfg, params_from_flat(cfg, params));
    });
}

/// load_checkpoint; cfg_out = {H, L, K, D} and rc, params (capacity from param_count).
LREF_API int lref_checkpoint_load(const char* path, int32_t* cfg_out, double* rc, double* params, int64_t cap) {
    return guarded([&] {
        const auto ck = lamm::model::load_checkpoint(path);
        cfg_out[0] = ck.config.hidden, cfg_out[1] = ck.config.layers, cfg_out[2] = ck.config.rbf;
        cfg_out[3] = ck.config.heads;
        *rc = ck.config.cutoff;
        if (static_cast<int64_t>(lamm::model::param_count(ck.params)) > cap) throw lamm::InputError("capacity");
        params_to_flat(ck.params, params);
    });
}

// ---- data layer (S/dataset.cpp:85-111, S/loss.cpp:17-111, S/trainer.cpp:82-100,
// S/model.cpp:195-202): checkers for paper_2505_22208_b200/csrc/host_data.cpp ----
LREF_API int lref_split_train_val(int64_t n, double val_fraction, uint64_t seed, int64_t* train, int64_t* n_train,
                                  int64_t* val, int64_t* n_val) {
    return guarded([&] {
        const auto s = lamm::dataset::split_train_val(static_cast<std::size_t>(n), val_fraction, seed);
        for (std::size_t k = 0; k < s.train.size(); ++k) train[k] = static_cast<int64_t>(s.train[k]);
        for (std::size_t k = 0; k < s.val.size(); ++k) val[k] = static_cast<int64_t>(s.val[k]);
        *n_train = static_cast<int64_t>(s.train.size());
        *n_val = static_cast<int64_t>(s.val.size());
    });
}

/// fit_normalizer over the batch's samples (this build's Eigen is oracle/shim:
/// its minimum-norm solve is a Jacobi pseudo-inverse, parity-unpinned).
LREF_API int lref_fit_normalizer(int32_t B, const int64_t* atom_ptr, const double* pos, const int32_t* Z,
                                 const uint8_t* emask, const uint8_t* fmask, const double* energy,
                                 const double* forces, double pseudo_std, double* rho, uint8_t* rho_has,
                                 double* stats /* mean, std, fstd, has */) {
    return guarded([&] {
        std::vector<lamm::Sample> pool;
        for (int s = 0; s < B; ++s) pool.push_back(sample_at(atom_ptr, pos, Z, nullptr, emask, fmask, energy, forces, s));
        const auto n = lamm::loss::fit_normalizer(pool, pseudo_std);
        for (int z = 0; z < 119; ++z) rho[z] = 0.0, rho_has[z] = 0;
        for (const auto& [z, v] : n.reference_energies) rho[z] = v, rho_has[z] = 1;
        stats[0] = n.energy_mean, stats[1] = n.energy_std, stats[2] = n.force_std;
        stats[3] = n.has_energy_stats ? 1.0 : 0.0;
    });
}

/// estimate_pseudo_force_std (S/trainer.cpp:82-100, file-local there): restated over
/// the reference's own apply_noise with the reference's probe seeds.
LREF_API int lref_pseudo_force_std(int32_t B, const int64_t* atom_ptr, const double* pos, const int32_t* Z,
                                   double sigma, int scheme, uint64_t seed, double* out) {
    return guarded([&] {
        constexpr uint64_t kProbeTag = 0x50535444;
        const int64_t probe = std::min<int64_t>(B, 256);
        double sum = 0.0, sq = 0.0;
        std::size_t count = 0;
        for (int64_t v = 0; v < probe; ++v) {
            lamm::denoise::NoiseConfig nc;
            nc.sigma = sigma;
            nc.scheme = scheme ? lamm::denoise::Scheme::centered : lamm::denoise::Scheme::baseline;
            nc.seed = lamm::mix_seed(seed, kProbeTag + static_cast<uint64_t>(v));
            const auto r = lamm::denoise::apply_noise(system_at(atom_ptr, pos, Z, static_cast<int>(v)), nc);
            for (const auto& f : r.pseudo_forces)
                for (double c : f) sum += c, sq += c * c, ++count;
        }
        if (count == 0) {
            *out = sigma;
            return;
        }
        const double mean = sum / static_cast<double>(count);
        *out = std::max(std::sqrt(std::max(sq / static_cast<double>(count) - mean * mean, 0.0)), 1e-8);
    });
}

LREF_API int lref_reset_heads(int H, int L, int K, double rc, int D, const double* params, int new_heads,
                              uint64_t seed, double* energy_head, double* force_head) {
    return guarded([&] {
        const auto cfg = make_cfg(H, L, K, rc, D);
        const auto p = lamm::model::reset_heads(params_from_flat(cfg, params), cfg, new_heads, seed);
        std::copy(p.energy_head.data(), p.energy_head.data() + p.energy_head.size(), energy_head);
        std::copy(p.force_head.data(), p.force_head.data() + p.force_head.size(), force_head);
    });
}

// ---- simulator (S/simulator.cpp:19-59): checker for lamm_simulate ----
LREF_API int lref_simulate(const int64_t* worker_atoms, int64_t n_batches, int G, int64_t samples_per_batch,
                           const double* cost4, double* step_time, double* step_idle, int32_t* step_realloc,
                           int64_t* step_max_atoms, double* worker_idle, double* totals4) {
    return guarded([&] {
        lamm::scheduler::MiniBatchSchedule sch;
        sch.workers = G;
        for (int64_t b = 0; b < n_batches; ++b) {
            lamm::scheduler::MiniBatch mb;
            mb.samples.resize(static_cast<std::size_t>(samples_per_batch));
            mb.worker_atoms.assign(worker_atoms + b * G, worker_atoms + (b + 1) * G);
            sch.batches.push_back(std::move(mb));
        }
        lamm::simulator::CostModel cm;
        cm.alpha_s = cost4[0], cm.beta_s_per_atom = cost4[1], cm.gamma_s = cost4[2], cm.delta_s = cost4[3];
        const auto r = lamm::simulator::simulate(sch, cm);
        for (std::size_t b = 0; b < r.steps.size(); ++b) {
            step_time[b] = r.steps[b].time_s;
            step_idle[b] = r.steps[b].idle_s;
            step_realloc[b] = r.steps[b].realloc_events;
            step_max_atoms[b] = r.steps[b].max_worker_atoms;
        }
        for (int g = 0; g < G; ++g) worker_idle[g] = r.worker_idle_s[static_cast<std::size_t>(g)];
        totals4[0] = r.total_s, totals4[1] = r.throughput_samples_per_s;
        totals4[2] = static_cast<double>(r.realloc_events), totals4[3] = static_cast<double>(r.samples);
    });
}
