// lamm_b200_trainer.hpp - the reference's training orchestration with the step
// body on the GPU.
//
//   lamm::trainer::pretrain       H/trainer.hpp:94-97,  S/trainer.cpp:384-413
//   lamm::trainer::finetune       H/trainer.hpp:108-111, S/trainer.cpp:415-443
//   lamm::trainer::denoise_bench  H/trainer.hpp:124-127, S/trainer.cpp:445-489
//
// Same signatures as the reference (plus an optional CUDA device ordinal), same
// result types, same seed streams, sinks, metric points and cadences. What runs
// where:
//
//   data layer (filter/split, mix plan, normalizer fit, noise, reset_heads,
//   config validation)
//        this library's native host code (csrc/host_data.cpp, host_sched.cpp):
//        lamm_filter_max_atoms, lamm_split_train_val, lamm_pseudo_force_std,
//        lamm_fit_normalizer, lamm_apply_noise, lamm_temperature_counts,
//        lamm_init_heads; the file-local glue of S/trainer.cpp (make_view,
//        build_refs, build_val_samples) is restated here over them. Only the
//        caller's value types (Catalog, Subset, Sample, TrainConfig, ...) come
//        from <lamm/...> headers: no reference function runs in this header
//   seed streams (mix_seed), epoch index, balanced schedule, init_params
//        this library's native host code (bit-exact with the reference)
//   step body (S/trainer.cpp:258-327): denoise -> normalize -> neighbour list
//        -> forward -> per-worker masked loss -> backward -> worker-order fp64
//        gradient sum -> /G -> norm -> clip -> RMS step
//        lamm_train_step_workers: one device, G simulated workers, parameters
//        and RMS state resident in HBM for the whole run
//   train batch stats at emit steps, validation (S/trainer.cpp:294-316, 491-553)
//        lamm_evaluate on the device (pre-update parameters for the batch stats)
//
// Parameters are read back to the host only for the checkpoint sink and the
// final result. Numbers are fp32 device arithmetic against the reference's
// fp64: trajectories agree to the step tolerance, not bit-for-bit
// (tests/cpp/test_trainer.cpp pins how closely).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <string>
#include <utility>
#include <vector>

#include "lamm_b200.hpp"

namespace lamm_b200::trainer {

// The reference's seed-stream tags (S/trainer.cpp:18-25): every random decision
// is mix_seed(cfg.seed, tag [+ k]), so a run here draws the same splits, epochs,
// schedules and noise as the reference run with the same seed.
enum : uint64_t {
    kInitStream = 0x1217,
    kHeadStream = 0xf1e7,
    kSplitStream = 0x53504c54,
    kEpochStream = 0x45504f43,
    kScheduleStream = 0x53434845,
    kNoiseStream = 0x4e4f4953,
    kValNoiseStream = 0x56414c4e,
    kProbeStream = 0x50535444,
};

namespace detail {

using Nan = std::numeric_limits<double>;

// lamm::trainer::validate_train_config (S/trainer.cpp:347-364) and
// lamm::model::validate_config (S/model.cpp:114-120), restated: the same checks and messages.
inline void check_train_config(const lamm::trainer::TrainConfig& cfg) {
    auto need = [](bool ok, const char* msg) {
        if (!ok) throw lamm::InputError(msg);
    };
    need(cfg.max_steps >= 1, "train: max_steps must be >= 1");
    need(cfg.learning_rate > 0.0, "train: learning_rate must be positive");
    need(cfg.clip_norm >= 0.0, "train: clip_norm must be >= 0");
    need(cfg.val_every >= 1, "train: val_every must be >= 1");
    need(cfg.checkpoint_every >= 0, "train: checkpoint_every must be >= 0");
    need(cfg.lambda_energy >= 0.0 && cfg.lambda_force >= 0.0, "train: lambdas must be >= 0");
    need(cfg.val_fraction >= 0.0 && cfg.val_fraction < 1.0, "train: val_fraction must be in [0, 1)");
    need(cfg.max_atoms >= 1, "train: max_atoms must be >= 1");
    need(cfg.noise_sigma > 0.0, "train: noise_sigma must be positive");
    need(cfg.energy_threshold >= 0.0 && cfg.force_threshold >= 0.0, "train: thresholds must be >= 0");
    need(cfg.rms_decay >= 0.0 && cfg.rms_decay < 1.0, "train: rms_decay must be in [0, 1)");
    need(cfg.rms_epsilon > 0.0, "train: rms_epsilon must be positive");
}
inline void check_model_config(const lamm::model::ModelConfig& c) {
    if (c.hidden < 1) throw lamm::InputError("model: hidden must be >= 1");
    if (c.layers < 0) throw lamm::InputError("model: layers must be >= 0");
    if (c.rbf < 2) throw lamm::InputError("model: rbf must be >= 2");
    if (!(c.cutoff > 0.0)) throw lamm::InputError("model: cutoff must be positive");
    if (c.heads < 1) throw lamm::InputError("model: heads must be >= 1");
}

// Packed (CSR) views of a subset's samples for the native data-layer calls.
template <class Samples>
inline PackedBatch pack_samples(const Samples& samples, const std::vector<int64_t>* ids = nullptr) {
    PackedBatch p;
    const size_t n = ids ? ids->size() : samples.size();
    for (size_t k = 0; k < n; ++k) p.add_sample(samples[ids ? static_cast<size_t>((*ids)[k]) : k]);
    return p;
}

inline int scheme_of(const lamm::trainer::TrainConfig& cfg) {
    return cfg.noise_scheme == lamm::denoise::Scheme::centered ? 1 : 0;
}

// make_denoising_sample (S/denoise.cpp:42-53) through the native apply_noise.
inline lamm::Sample denoising_copy(const lamm::Sample& src, const lamm::trainer::TrainConfig& cfg, uint64_t seed,
                                   int dataset_index, int subset_id) {
    const size_t n = src.system.positions.size();
    std::vector<double> pos(3 * n), noisy(3 * n), pf(3 * n);
    for (size_t a = 0; a < n; ++a)
        for (int c = 0; c < 3; ++c) pos[3 * a + c] = src.system.positions[a][c];
    check(lamm_apply_noise(pos.data(), static_cast<int64_t>(n), cfg.noise_sigma, scheme_of(cfg), seed, noisy.data(),
                           pf.data()));
    lamm::Sample out;
    out.system = src.system;
    out.labels.forces.resize(n);
    for (size_t a = 0; a < n; ++a)
        for (int c = 0; c < 3; ++c) {
            out.system.positions[a][c] = noisy[3 * a + c];
            out.labels.forces[a][c] = pf[3 * a + c];
        }
    out.labels.force_mask = true;
    out.labels.energy_mask = false;
    out.labels.dataset_index = dataset_index;
    out.subset_id = subset_id;
    return out;
}

// A subset resolved for training: kept sample ids split into train / val.
struct Split {
    const lamm::dataset::Subset* subset = nullptr;
    std::vector<int64_t> train, val;
    bool denoising = false;
};

inline Split split_subset(const lamm::dataset::Subset& subset, const lamm::trainer::TrainConfig& cfg,
                          uint64_t seed) {
    Split s;
    s.subset = &subset;
    s.denoising = subset.meta.task == lamm::dataset::TaskKind::denoising;
    std::vector<int64_t> ptr{0};
    for (const auto& smp : subset.samples) ptr.push_back(ptr.back() + static_cast<int64_t>(smp.system.size()));
    const int64_t ns = static_cast<int64_t>(subset.samples.size());
    std::vector<int64_t> kept(static_cast<size_t>(std::max<int64_t>(ns, 1)));
    int64_t nk = 0;
    check(lamm_filter_max_atoms(ptr.data(), ns, cfg.max_atoms, kept.data(), &nk));
    if (nk == 0) throw lamm::InputError("subset \"" + subset.meta.name + "\": no samples under the atom limit");
    std::vector<int64_t> tr(static_cast<size_t>(nk)), va(static_cast<size_t>(nk));
    int64_t nt = 0, nv = 0;
    check(lamm_split_train_val(nk, cfg.val_fraction, seed, tr.data(), &nt, va.data(), &nv));
    s.train.reserve(static_cast<size_t>(nt));
    for (int64_t k = 0; k < nt; ++k) s.train.push_back(kept[static_cast<size_t>(tr[static_cast<size_t>(k)])]);
    for (int64_t k = 0; k < nv; ++k) s.val.push_back(kept[static_cast<size_t>(va[static_cast<size_t>(k)])]);
    if (s.train.empty()) throw lamm::InputError("subset \"" + subset.meta.name + "\": empty training split");
    return s;
}

inline const lamm::Sample& sample_of(const Split& s, int64_t train_pos) {
    return s.subset->samples[static_cast<size_t>(s.train[static_cast<size_t>(train_pos)])];
}

// Pseudo-force scale of a denoising subset: std of the noise labels over a
// fixed probe of up to 256 training structures (S/trainer.cpp:85-105).
inline double pseudo_force_scale(const Split& s, const lamm::trainer::TrainConfig& cfg) {
    const std::vector<int64_t> probe(s.train.begin(), s.train.begin() + std::min<size_t>(s.train.size(), 256));
    const PackedBatch p = pack_samples(s.subset->samples, &probe);
    double out = 0.0;
    check(lamm_pseudo_force_std(p.atom_ptr.data(), p.positions.data(), nullptr, static_cast<int64_t>(probe.size()),
                                cfg.noise_sigma, scheme_of(cfg), cfg.seed, &out));
    return out;
}

// loss::DatasetNormalizer from the native fit (rho by Z -> the reference's map).
inline lamm::loss::DatasetNormalizer normalizer_of(const lamm_normalizer& n) {
    lamm::loss::DatasetNormalizer d;
    for (int z = 0; z < 119; ++z)
        if (n.rho_has[z]) d.reference_energies[z] = n.rho[z];
    d.energy_mean = n.energy_mean;
    d.energy_std = n.energy_std;
    d.force_std = n.force_std;
    d.has_energy_stats = n.has_energy_stats != 0;
    return d;
}

// One normalizer per prediction channel over the pooled training samples of
// the subsets on that channel (S/trainer.cpp:107-131).
inline lamm::loss::ReferenceTable fit_channels(const std::vector<Split>& splits, int heads,
                                               const lamm::trainer::TrainConfig& cfg) {
    lamm::loss::ReferenceTable t;
    t.per_dataset.resize(static_cast<size_t>(heads));
    for (int d = 0; d < heads; ++d) {
        PackedBatch pool;
        double pseudo = 0.0;
        for (const auto& s : splits) {
            if (s.subset->meta.head_index != d) continue;
            if (s.denoising) {
                pseudo = std::max(pseudo, pseudo_force_scale(s, cfg));
            } else {
                for (const auto id : s.train) pool.add_sample(s.subset->samples[static_cast<size_t>(id)]);
            }
        }
        if (pool.size() > 0 || pseudo > 0.0) {
            lamm_normalizer n{};
            const lamm_batch_view v = pool.view();
            check(lamm_fit_normalizer(&v, pseudo, &n));
            t.per_dataset[static_cast<size_t>(d)] = normalizer_of(n);
        }
    }
    return t;
}

// Held-out samples; denoising subsets contribute one fixed noisy copy per
// structure when asked (S/trainer.cpp:133-156).
inline std::vector<lamm::Sample> held_out(const std::vector<Split>& splits, const lamm::trainer::TrainConfig& cfg,
                                          bool with_denoising) {
    std::vector<lamm::Sample> out;
    uint64_t ordinal = 0;
    for (const auto& s : splits) {
        for (const auto id : s.val) {
            const auto& raw = s.subset->samples[static_cast<size_t>(id)];
            if (!s.denoising) {
                out.push_back(raw);
            } else if (with_denoising) {
                out.push_back(denoising_copy(raw, cfg, lamm_mix_seed(cfg.seed, kValNoiseStream + ordinal),
                                             s.subset->meta.head_index, raw.subset_id));
            }
            ++ordinal;
        }
    }
    return out;
}

struct Run {
    std::vector<Split> splits;
    lamm::dataset::MixPlan mix;
    lamm::scheduler::ScheduleConfig sched;
    lamm::model::ModelConfig mcfg;
    lamm::trainer::TrainConfig cfg;
    lamm::loss::ReferenceTable refs;
    std::vector<lamm::Sample> val;
};

// One epoch's (subset, train position) draws through the native epoch index.
inline std::vector<std::pair<int, int64_t>> epoch_draws(const Run& run, uint64_t seed) {
    const int32_t k = static_cast<int32_t>(run.splits.size());
    if (run.mix.repeats.size() != run.splits.size()) throw lamm::InputError("mix plan length != subset count");
    std::vector<int64_t> sizes;
    int64_t cap = 0;
    for (int32_t i = 0; i < k; ++i) {
        sizes.push_back(static_cast<int64_t>(run.splits[static_cast<size_t>(i)].train.size()));
        cap += static_cast<int64_t>(std::llround(run.mix.repeats[static_cast<size_t>(i)])) + 1;
    }
    std::vector<int32_t> sub(static_cast<size_t>(cap));
    std::vector<int64_t> pos(static_cast<size_t>(cap));
    int64_t n = 0;
    check(lamm_build_epoch_index(run.mix.repeats.data(), sizes.data(), k, seed, cap, sub.data(), pos.data(), &n));
    std::vector<std::pair<int, int64_t>> out(static_cast<size_t>(n));
    for (int64_t e = 0; e < n; ++e) out[static_cast<size_t>(e)] = {sub[static_cast<size_t>(e)], pos[static_cast<size_t>(e)]};
    return out;
}

// run_loop (S/trainer.cpp:191-343) with the device step.
inline lamm::trainer::RunMetrics run(const Run& r, lamm::model::ModelParams& params, int device,
                                     const lamm::trainer::CheckpointSink& on_checkpoint,
                                     const lamm::trainer::PointSink& on_point) {
    const auto& cfg = r.cfg;
    check_train_config(cfg);
    check_model_config(r.mcfg);
    for (const auto& s : r.splits)
        if (s.subset->meta.head_index < 0 || s.subset->meta.head_index >= r.mcfg.heads)
            throw lamm::InputError("subset \"" + s.subset->meta.name + "\" trains head " +
                                   std::to_string(s.subset->meta.head_index) + " but the model has " +
                                   std::to_string(r.mcfg.heads));

    Device dev(r.mcfg, device);
    dev.set_params_from(params);
    dev.set_rms_state(std::vector<double>(dev.param_count(), 0.0));  // fresh RmsOptimizer (v = 0)
    dev.set_reference_table(r.refs);

    lamm::trainer::RunMetrics m;
    m.best_energy_mae = m.best_force_mae = m.final_loss = Nan::quiet_NaN();
    auto emit = [&](lamm::trainer::MetricPoint p) {
        if (on_point) on_point(p);
        m.points.push_back(std::move(p));
    };
    auto validate = [&](int64_t step) {
        if (r.val.empty()) return;
        const auto e = evaluate<lamm::trainer::EvalResult>(dev, std::span<const lamm::Sample>(r.val));
        emit({step, "val", e.energy_mae, e.force_mae, Nan::quiet_NaN()});
        if (!std::isnan(e.energy_mae) && !(m.best_energy_mae <= e.energy_mae)) m.best_energy_mae = e.energy_mae;
        if (!std::isnan(e.force_mae) && !(m.best_force_mae <= e.force_mae)) m.best_force_mae = e.force_mae;
        if (cfg.energy_threshold > 0.0 && m.steps_to_energy_threshold < 0 && e.energy_mae <= cfg.energy_threshold)
            m.steps_to_energy_threshold = step;
        if (cfg.force_threshold > 0.0 && m.steps_to_force_threshold < 0 && e.force_mae <= cfg.force_threshold)
            m.steps_to_force_threshold = step;
    };
    auto host_params = [&] {
        unflatten(dev.params(), params);
        return params;
    };

    const int G = r.sched.workers, B = r.sched.batch_per_worker;
    int64_t step = 0;
    for (int64_t epoch = 0; step < cfg.max_steps; ++epoch) {
        const auto draws = epoch_draws(r, lamm_mix_seed(cfg.seed, kEpochStream + static_cast<uint64_t>(epoch)));
        std::vector<int64_t> atoms(draws.size());
        for (size_t e = 0; e < draws.size(); ++e)
            atoms[e] = static_cast<int64_t>(
                sample_of(r.splits[static_cast<size_t>(draws[e].first)], draws[e].second).system.size());
        auto sc = r.sched;
        sc.seed = lamm_mix_seed(cfg.seed, kScheduleStream + static_cast<uint64_t>(epoch));
        const auto schedule = plan<lamm::scheduler::MiniBatchSchedule>(atoms, sc);
        if (schedule.batches.empty())
            throw lamm::InputError("schedule produced no mini-batches; reduce workers*batch_per_worker"
                                   " or num_splits, or provide more data");

        for (const auto& mb : schedule.batches) {
            if (step >= cfg.max_steps) break;
            std::vector<lamm::Sample> batch;
            std::vector<uint8_t> noisy;
            batch.reserve(static_cast<size_t>(G * B));
            for (int k = 0; k < G * B; ++k) {
                const auto& [si, tp] = draws[static_cast<size_t>(mb.samples[static_cast<size_t>(k)].sample)];
                const auto& s = r.splits[static_cast<size_t>(si)];
                batch.push_back(sample_of(s, tp));
                if (s.denoising) batch.back().labels.dataset_index = s.subset->meta.head_index;
                noisy.push_back(s.denoising ? 1 : 0);
            }
            const bool report = (step + 1) % cfg.val_every == 0 || step + 1 == cfg.max_steps;
            lamm::trainer::EvalResult stats{Nan::quiet_NaN(), Nan::quiet_NaN(), 0, 0};
            if (report) {  // batch stats of this step's predictions, physical units (S/trainer.cpp:294-316)
                std::vector<lamm::Sample> phys = batch;
                for (int k = 0; k < G * B; ++k) {
                    if (!noisy[static_cast<size_t>(k)]) continue;
                    // the draws the device step makes for worker slot k (S/trainer.cpp:276-277)
                    const auto& src = batch[static_cast<size_t>(k)];
                    phys[static_cast<size_t>(k)] = denoising_copy(
                        src, cfg,
                        lamm_mix_seed(lamm_mix_seed(cfg.seed, kNoiseStream + static_cast<uint64_t>(step)),
                                      static_cast<uint64_t>(k)),
                        src.labels.dataset_index, src.subset_id);
                }
                stats = evaluate<lamm::trainer::EvalResult>(dev, std::span<const lamm::Sample>(phys));
            }
            const StepResult res = train_step_workers(dev, std::span<const lamm::Sample>(batch),
                                                      std::span<const uint8_t>(noisy), cfg, step, G);
            ++step;
            m.final_loss = res.loss;
            const bool last = step == cfg.max_steps;
            if (report) {
                emit({step, "train", stats.energy_mae, stats.force_mae, res.loss});
                validate(step);
            }
            if (on_checkpoint && cfg.checkpoint_every > 0 && step % cfg.checkpoint_every == 0 && !last)
                on_checkpoint(step, r.mcfg, host_params(), r.refs);
        }
    }
    host_params();
    if (on_checkpoint) on_checkpoint(step, r.mcfg, params, r.refs);
    return m;
}

// init_params of the config into freshly shaped tensors (H/model.hpp:46-52 shapes).
inline lamm::model::ModelParams initial_params(const lamm::model::ModelConfig& c, uint64_t seed) {
    const auto H = static_cast<size_t>(c.hidden), K = static_cast<size_t>(c.rbf), D = static_cast<size_t>(c.heads);
    lamm::model::ModelParams p;
    p.embedding = lamm::Matrix(118, H);
    p.filter.assign(static_cast<size_t>(c.layers), lamm::Matrix(H, K));
    p.update.assign(static_cast<size_t>(c.layers), lamm::Matrix(H, H));
    p.energy_head = lamm::Matrix(H, D);
    p.force_head = lamm::Matrix(2 * H + K, D);
    init_params(p, c, seed);
    return p;
}

inline void single_subset_mix(Run& r) {
    r.mix.temperature = 1.0;
    r.mix.repeats = {static_cast<double>(r.splits.front().train.size())};
}

}  // namespace detail

// lamm::trainer::pretrain: 300-atom filter, train/val split, per-channel
// normalizer fit, temperature-sampled epochs, balanced schedule, device steps.
inline lamm::trainer::PretrainResult pretrain(const lamm::dataset::Catalog& catalog,
                                              const lamm::dataset::MixPlan& mix,
                                              const lamm::scheduler::ScheduleConfig& sched,
                                              const lamm::model::ModelConfig& model_cfg,
                                              const lamm::trainer::TrainConfig& cfg,
                                              const lamm::trainer::CheckpointSink& on_checkpoint = {},
                                              const lamm::trainer::PointSink& on_point = {}, int device = 0) {
    if (catalog.subsets.empty()) throw lamm::InputError("pretrain: catalog has no subsets");
    if (!mix.repeats.empty() && mix.repeats.size() != catalog.subsets.size())
        throw lamm::InputError("pretrain: mix plan length != subset count");
    detail::Run r;
    r.sched = sched;
    r.mcfg = model_cfg;
    r.cfg = cfg;
    for (size_t k = 0; k < catalog.subsets.size(); ++k)
        r.splits.push_back(detail::split_subset(catalog.subsets[k], cfg, lamm_mix_seed(cfg.seed, kSplitStream + k)));
    r.refs = detail::fit_channels(r.splits, model_cfg.heads, cfg);
    if (mix.repeats.empty()) {
        std::vector<double> sizes;
        for (const auto& s : r.splits) sizes.push_back(static_cast<double>(s.train.size()));
        r.mix.temperature = mix.temperature;  // dataset::make_mix_plan (S/dataset.cpp:54-59)
        r.mix.repeats.assign(sizes.size(), 0.0);
        check(lamm_temperature_counts(sizes.data(), static_cast<int32_t>(sizes.size()), mix.temperature,
                                      r.mix.repeats.data()));
    } else {
        r.mix = mix;
    }
    r.val = detail::held_out(r.splits, cfg, false);

    lamm::trainer::PretrainResult out;
    out.config = model_cfg;
    out.params = detail::initial_params(model_cfg, lamm_mix_seed(cfg.seed, kInitStream));
    out.refs = r.refs;
    out.metrics = detail::run(r, out.params, device, on_checkpoint, on_point);
    return out;
}

// lamm::trainer::finetune: one fresh head, the encoder from the checkpoint,
// references refit on the target's training split.
inline lamm::trainer::FinetuneResult finetune(const lamm::model::Checkpoint& start,
                                              const lamm::dataset::Subset& target,
                                              const lamm::scheduler::ScheduleConfig& sched,
                                              const lamm::trainer::TrainConfig& cfg,
                                              const lamm::trainer::CheckpointSink& on_checkpoint = {},
                                              const lamm::trainer::PointSink& on_point = {}, int device = 0) {
    detail::check_model_config(start.config);
    lamm::dataset::Subset local = target;
    local.meta.head_index = 0;
    for (auto& s : local.samples) s.labels.dataset_index = 0;

    detail::Run r;
    r.sched = sched;
    r.mcfg = start.config;
    r.mcfg.heads = 1;
    r.cfg = cfg;
    r.splits.push_back(detail::split_subset(local, cfg, lamm_mix_seed(cfg.seed, kSplitStream)));
    r.refs = detail::fit_channels(r.splits, 1, cfg);
    detail::single_subset_mix(r);
    r.val = detail::held_out(r.splits, cfg, true);

    lamm::trainer::FinetuneResult out;
    out.config = r.mcfg;
    out.params = start.params;  // model::reset_heads (S/model.cpp:195-202): one fresh head, natively drawn
    {
        const auto H = static_cast<size_t>(start.config.hidden), K = static_cast<size_t>(start.config.rbf);
        lamm_model_config mc{start.config.hidden, start.config.layers, start.config.rbf, 1, start.config.cutoff};
        out.params.energy_head = lamm::Matrix(H, 1);
        out.params.force_head = lamm::Matrix(2 * H + K, 1);
        check(lamm_init_heads(&mc, 1, lamm_mix_seed(cfg.seed, kHeadStream), out.params.energy_head.data(),
                              out.params.force_head.data()));
    }
    out.refs = r.refs;
    out.metrics = detail::run(r, out.params, device, on_checkpoint, on_point);
    return out;
}

// lamm::trainer::denoise_bench: baseline vs centered labels, identical seeds,
// data and noise draws; steps to the pseudo-force MAE threshold.
inline lamm::trainer::DenoiseBenchResult denoise_bench(const lamm::dataset::Subset& unlabeled,
                                                       const lamm::scheduler::ScheduleConfig& sched,
                                                       const lamm::model::ModelConfig& model_cfg,
                                                       const lamm::trainer::TrainConfig& cfg, double threshold_mae,
                                                       const lamm::trainer::PointSink& on_point = {},
                                                       int device = 0) {
    if (!(threshold_mae >= 0.0)) throw lamm::InputError("denoise_bench: threshold must be >= 0");
    lamm::dataset::Subset local = unlabeled;
    local.meta.task = lamm::dataset::TaskKind::denoising;
    local.meta.head_index = 0;
    for (auto& s : local.samples) {
        s.labels = lamm::Labels{};
        s.labels.dataset_index = 0;
    }
    lamm::model::ModelConfig mcfg = model_cfg;
    mcfg.heads = 1;
    const auto initial = detail::initial_params(mcfg, lamm_mix_seed(cfg.seed, kInitStream));

    lamm::trainer::DenoiseBenchResult out;
    out.threshold = threshold_mae;
    for (const auto scheme : {lamm::denoise::Scheme::baseline, lamm::denoise::Scheme::centered}) {
        detail::Run r;
        r.sched = sched;
        r.mcfg = mcfg;
        r.cfg = cfg;
        r.cfg.noise_scheme = scheme;
        r.cfg.force_threshold = threshold_mae;
        r.splits.push_back(detail::split_subset(local, r.cfg, lamm_mix_seed(cfg.seed, kSplitStream)));
        r.refs = detail::fit_channels(r.splits, 1, r.cfg);
        detail::single_subset_mix(r);
        r.val = detail::held_out(r.splits, r.cfg, true);
        auto params = initial;
        auto metrics = detail::run(r, params, device, {}, on_point);
        if (scheme == lamm::denoise::Scheme::baseline) {
            out.baseline_steps_to_threshold = metrics.steps_to_force_threshold;
            out.baseline = std::move(metrics);
        } else {
            out.centered_steps_to_threshold = metrics.steps_to_force_threshold;
            out.centered = std::move(metrics);
        }
    }
    return out;
}

}  // namespace lamm_b200::trainer
