// test_dropin.cpp - the C++ drop-in check: include/lamm_b200.hpp driven with
// the REFERENCE's own types (lamm::AtomicSystem, lamm::Sample,
// lamm::model::ModelParams / Prediction, lamm::NeighborList,
// lamm::scheduler::MiniBatchSchedule ...) and compared with the reference
// functions it replaces, called in the same binary.
//
// Test infrastructure: built by oracle/Makefile (target `dropin`) from the
// reference sources under /root/reference (never copied) into
// oracle/_ref/test_dropin, linked against the product library
// paper_2505_22208_b200/liblamm_b200.so; run by tests/test_cxx_dropin.py on a
// GPU. Prints one line per check and exits non-zero on any failure.
//
// Bars (SURVEY.md §8 parity contract): neighbour lists and schedules
// bit-exact; energies, forces, loss gradients and every parameter-gradient
// tensor within 1e-4 relative (both max|d|/max|ref| and ||d||/||ref||).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "lamm/core.hpp"
#include "lamm/dataset.hpp"
#include "lamm/denoise.hpp"
#include "lamm/loss.hpp"
#include "lamm/model.hpp"
#include "lamm/rng.hpp"
#include "lamm/scheduler.hpp"
#include "lamm/trainer.hpp"
#include "lamm_b200.hpp"

namespace {

int g_failures = 0;
constexpr double kTol = 1e-4;

void report(bool ok, const std::string& what, const std::string& detail = "") {
    std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", what.c_str(), detail.empty() ? "" : "  ", detail.c_str());
    if (!ok) ++g_failures;
}

// max(max|a-b| / max|b|, ||a-b|| / ||b||)
double rel(const double* a, const double* b, size_t n) {
    double dmax = 0, rmax = 0, d2 = 0, r2 = 0;
    for (size_t k = 0; k < n; ++k) {
        const double d = a[k] - b[k];
        dmax = std::max(dmax, std::abs(d));
        rmax = std::max(rmax, std::abs(b[k]));
        d2 += d * d;
        r2 += b[k] * b[k];
    }
    if (rmax == 0) return dmax == 0 ? 0 : INFINITY;
    return std::max(dmax / rmax, std::sqrt(d2 / r2));
}
double rel(const std::vector<double>& a, const std::vector<double>& b) {
    if (a.size() != b.size()) return INFINITY;
    return rel(a.data(), b.data(), a.size());
}

std::string fmt(double x) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "rel=%.3g", x);
    return buf;
}

std::vector<double> concat_energy(const std::vector<lamm::model::Prediction>& p) {
    std::vector<double> out;
    for (const auto& x : p) out.insert(out.end(), x.energy.begin(), x.energy.end());
    return out;
}
std::vector<double> concat_forces(const std::vector<lamm::model::Prediction>& p) {
    std::vector<double> out;
    for (const auto& x : p) out.insert(out.end(), x.forces.begin(), x.forces.end());
    return out;
}

lamm::loss::ReferenceTable make_table(int D) {
    lamm::loss::ReferenceTable t;
    t.per_dataset.resize(static_cast<size_t>(D));
    for (int d = 0; d < D; ++d) {
        auto& n = t.per_dataset[static_cast<size_t>(d)];
        n.reference_energies = {{1, -0.45 - 0.01 * d}, {6, -1.2}, {7, -0.9 + 0.02 * d}, {8, -1.05}};
        n.energy_mean = 0.3 - 0.1 * d;
        n.energy_std = 1.7 + 0.2 * d;
        n.force_std = 1.3 + 0.1 * d;
        n.has_energy_stats = true;
    }
    return t;
}

std::vector<lamm::Sample> make_samples(int count, int D, uint64_t seed) {
    lamm::dataset::SynthSpec spec;
    spec.elements = {1, 6, 7, 8};
    spec.atom_count_mode = 20.0;
    spec.atom_count_sigma = 0.5;
    spec.min_atoms = 2;
    spec.max_atoms = 60;
    auto samples = lamm::dataset::synth_generate(spec, count, seed);
    for (size_t s = 0; s < samples.size(); ++s) {
        auto& l = samples[s].labels;
        l.dataset_index = static_cast<int>(s) % D;
        if (s % 5 == 1) l.energy_mask = false;  // label present but masked out
        if (s % 7 == 2) l.force_mask = false;
    }
    return samples;
}

void check_neighbor_lists(lamm_b200::Device& dev, const std::vector<lamm::Sample>& samples, double rc) {
    std::vector<lamm::AtomicSystem> systems;
    for (const auto& s : samples) systems.push_back(s.system);
    // a sample whose atoms are all farther apart than rc and an isolated atom
    systems.push_back(lamm::AtomicSystem{{{0, 0, 0}, {0, 0, 6.0}, {0, 7.5, 0}}, {1, 6, 8}});
    systems.push_back(lamm::AtomicSystem{{{1, 2, 3}}, {6}});
    const auto ours = lamm_b200::build_neighbor_lists<lamm::NeighborList>(
        dev, std::span<const lamm::AtomicSystem>(systems), rc);
    bool ok = ours.size() == systems.size();
    size_t pairs = 0;
    for (size_t s = 0; ok && s < systems.size(); ++s) {
        const auto ref = lamm::build_neighbor_list(systems[s], rc);
        ok = ref.pairs.size() == ours[s].pairs.size() && ours[s].cutoff == ref.cutoff;
        for (size_t p = 0; ok && p < ref.pairs.size(); ++p) {
            const auto &a = ours[s].pairs[p], &b = ref.pairs[p];
            ok = a.i == b.i && a.j == b.j && std::memcmp(&a.distance, &b.distance, 8) == 0 &&
                 std::memcmp(a.unit.data(), b.unit.data(), 24) == 0;
        }
        pairs += ref.pairs.size();
    }
    report(ok, "build_neighbor_list bit-exact (i, j, distance, unit)", std::to_string(pairs) + " pairs");
    const auto one = lamm_b200::build_neighbor_list<lamm::NeighborList>(dev, systems[0], rc);
    const auto ref0 = lamm::build_neighbor_list(systems[0], rc);
    report(one.pairs.size() == ref0.pairs.size(), "build_neighbor_list single-system signature");
}

void check_model(lamm_b200::Device& dev, const std::vector<lamm::Sample>& samples,
                 const lamm::model::ModelConfig& cfg, const lamm::model::ModelParams& params,
                 const lamm::loss::ReferenceTable& table) {
    // reference: normalize -> forward(cache) -> masked_loss_grad -> backward
    std::vector<lamm::Sample> normalized;
    std::vector<lamm::model::ForwardCache> caches(samples.size());
    std::vector<lamm::model::Prediction> ref_pred;
    for (size_t s = 0; s < samples.size(); ++s) {
        normalized.push_back(lamm::loss::normalize_labels(samples[s], table));
        ref_pred.push_back(lamm::model::forward(normalized.back().system, params, cfg, &caches[s]));
    }
    const lamm::loss::LossConfig lcfg{1.0, 1.3};
    std::vector<lamm::model::PredictionGrad> ref_pg;
    const auto ref_loss = lamm::loss::masked_loss_grad(normalized, ref_pred, lcfg, ref_pg);
    auto ref_grads = lamm::model::zero_like(params);
    for (size_t s = 0; s < samples.size(); ++s) lamm::model::backward(caches[s], params, cfg, ref_pg[s], ref_grads);

    // device: raw samples, normalize_labels runs on the device
    dev.set_reference_table(table);
    lamm_b200::DeviceCache cache;
    const auto pred = lamm_b200::forward_samples<lamm::model::Prediction>(
        dev, std::span<const lamm::Sample>(samples), params, cfg, &cache);
    report(rel(concat_energy(pred), concat_energy(ref_pred)) <= kTol, "forward energies",
           fmt(rel(concat_energy(pred), concat_energy(ref_pred))));
    report(rel(concat_forces(pred), concat_forces(ref_pred)) <= kTol, "forward forces",
           fmt(rel(concat_forces(pred), concat_forces(ref_pred))));
    bool shapes = true;
    for (size_t s = 0; s < samples.size(); ++s)
        shapes &= pred[s].n_atoms == ref_pred[s].n_atoms && pred[s].heads == ref_pred[s].heads;
    report(shapes, "Prediction n_atoms / heads");

    std::vector<lamm::model::PredictionGrad> pg;
    const auto loss = lamm_b200::masked_loss_grad<lamm::loss::LossBreakdown>(dev, cache, lcfg, pg);
    const double lrel = std::abs(loss.total - ref_loss.total) / std::abs(ref_loss.total);
    report(lrel <= kTol && loss.energy_labeled == ref_loss.energy_labeled &&
               loss.force_labeled == ref_loss.force_labeled && loss.energy_empty == ref_loss.energy_empty &&
               loss.force_empty == ref_loss.force_empty,
           "masked_loss_grad breakdown", fmt(lrel));
    report(rel(concat_energy(pg), concat_energy(ref_pg)) <= kTol, "masked_loss_grad dL/dE",
           fmt(rel(concat_energy(pg), concat_energy(ref_pg))));
    report(rel(concat_forces(pg), concat_forces(ref_pg)) <= kTol, "masked_loss_grad dL/dF",
           fmt(rel(concat_forces(pg), concat_forces(ref_pg))));

    // backward with the reference's upstream gradients, accumulate semantics
    auto grads = lamm::model::zero_like(params);
    lamm_b200::backward(dev, cache, params, cfg, std::span<const lamm::model::PredictionGrad>(ref_pg), grads);
    std::vector<const lamm::Matrix*> mine, theirs;
    lamm::model::for_each_tensor(grads, [&](const lamm::Matrix& m) { mine.push_back(&m); });
    lamm::model::for_each_tensor(ref_grads, [&](const lamm::Matrix& m) { theirs.push_back(&m); });
    const char* names[] = {"embedding", "filter", "update", "energy_head", "force_head"};
    for (size_t t = 0; t < mine.size(); ++t) {
        const int L = cfg.layers;
        const int kind = t == 0 ? 0 : t <= static_cast<size_t>(L) ? 1 : t <= static_cast<size_t>(2 * L) ? 2 : t == mine.size() - 2 ? 3 : 4;
        const double r = rel(mine[t]->data(), theirs[t]->data(), theirs[t]->size());
        report(r <= kTol, std::string("backward d/d") + names[kind] + "[" + std::to_string(t) + "]", fmt(r));
    }
    lamm_b200::backward(dev, cache, params, cfg, std::span<const lamm::model::PredictionGrad>(ref_pg), grads);
    auto twice = ref_grads;
    lamm::model::scale_params(twice, 2.0);
    const auto a = lamm_b200::flatten(grads), b = lamm_b200::flatten(twice);
    report(rel(a, b) <= kTol, "backward accumulates (+=) into Gradients", fmt(rel(a, b)));
}

void check_scheduler() {
    const std::vector<int64_t> small{8, 7, 2, 1};
    const auto w = lamm_b200::greedy_assign(small, 2, 2);
    report(w == lamm::scheduler::greedy_assign(small, 2, 2) && w == std::vector<int>{0, 1, 1, 0},
           "greedy_assign({8,7,2,1}, 2, 2) == {0,1,1,0}");
    lamm::Rng rng(17);
    std::vector<int64_t> atoms(5000);
    for (auto& a : atoms) a = 2 + static_cast<int64_t>(std::exp(3.0 + 1.0 * rng.normal())) % 1999;
    using lamm::scheduler::Mode;
    for (Mode mode : {Mode::balanced, Mode::greedy_only, Mode::naive}) {
        lamm::scheduler::ScheduleConfig cfg{8, 4, 100, 3, mode};
        const auto ref = lamm::scheduler::plan(atoms, cfg);
        const auto ours = lamm_b200::plan<lamm::scheduler::MiniBatchSchedule>(atoms, cfg);
        bool ok = ref.batches.size() == ours.batches.size() && ref.dropped_samples == ours.dropped_samples &&
                  ref.workers == ours.workers && ref.batch_per_worker == ours.batch_per_worker;
        for (size_t s = 0; ok && s < ref.batches.size(); ++s) {
            ok = ref.batches[s].worker_atoms == ours.batches[s].worker_atoms &&
                 ref.batches[s].samples.size() == ours.batches[s].samples.size();
            for (size_t k = 0; ok && k < ref.batches[s].samples.size(); ++k) {
                const auto &x = ref.batches[s].samples[k], &y = ours.batches[s].samples[k];
                ok = x.sample == y.sample && x.worker == y.worker && x.atoms == y.atoms && x.split == y.split &&
                     x.chunk_rank == y.chunk_rank;
            }
        }
        report(ok, "plan bit-exact, mode " + lamm::scheduler::to_string(mode),
               std::to_string(ref.batches.size()) + " mini-batches");
    }
}

// Replica of the run_loop step body (S/trainer.cpp:258-327) for G = 1 with a
// denoising sample every third position, against lamm_b200::train_step.
void check_train_step(const std::vector<lamm::Sample>& samples, const lamm::model::ModelConfig& cfg,
                      const lamm::model::ModelParams& params0, const lamm::loss::ReferenceTable& table) {
    const uint64_t seed = 1234;
    const int64_t step = 3;
    const double sigma = 0.3, lr = 1e-3, decay = 0.99, eps = 1e-8;
    std::vector<uint8_t> denoise(samples.size());
    std::vector<lamm::Sample> normalized;
    std::vector<lamm::model::ForwardCache> caches(samples.size());
    std::vector<lamm::model::Prediction> preds;
    for (size_t b = 0; b < samples.size(); ++b) {
        denoise[b] = b % 3 == 0;
        lamm::Sample raw = samples[b];
        if (denoise[b]) {
            lamm::denoise::NoiseConfig n{sigma, lamm::denoise::Scheme::centered,
                                         lamm::mix_seed(lamm::mix_seed(seed, 0x4e4f4953 + step), b)};
            raw = lamm::denoise::make_denoising_sample(samples[b].system, n, samples[b].labels.dataset_index,
                                                       samples[b].subset_id);
        }
        normalized.push_back(lamm::loss::normalize_labels(raw, table));
        preds.push_back(lamm::model::forward(normalized.back().system, params0, cfg, &caches[b]));
    }
    std::vector<lamm::model::PredictionGrad> pg;
    const auto br = lamm::loss::masked_loss_grad(normalized, preds, lamm::loss::LossConfig{}, pg);
    auto grads = lamm::model::zero_like(params0);
    for (size_t b = 0; b < samples.size(); ++b) lamm::model::backward(caches[b], params0, cfg, pg[b], grads);
    const double gnorm = lamm::model::global_norm(grads);
    std::vector<double> g = lamm_b200::flatten(grads), v(g.size());
    for (size_t k = 0; k < g.size(); ++k) v[k] = (1.0 - decay) * g[k] * g[k];  // v0 = 0

    lamm_b200::Device dev(cfg, 0);
    dev.set_params_from(params0);
    dev.set_rms_state(std::vector<double>(g.size(), 0.0));
    dev.set_reference_table(table);
    struct {
        double learning_rate = 1e-3, clip_norm = 1e9, rms_decay = 0.99, rms_epsilon = 1e-8, noise_sigma = 0.3;
        lamm::denoise::Scheme noise_scheme = lamm::denoise::Scheme::centered;
        uint64_t seed = 1234;
        double lambda_energy = 1.0, lambda_force = 1.0;
    } tcfg;
    (void)lr;
    (void)eps;
    const auto r = lamm_b200::train_step(dev, std::span<const lamm::Sample>(samples),
                                         std::span<const uint8_t>(denoise), tcfg, step, 1, 0);
    report(std::abs(r.loss - br.total) <= kTol * std::abs(br.total), "train_step loss (denoise + labelled)",
           fmt(std::abs(r.loss - br.total) / std::abs(br.total)));
    report(std::abs(r.grad_norm - gnorm) <= kTol * gnorm, "train_step grad_norm",
           fmt(std::abs(r.grad_norm - gnorm) / gnorm));
    report(rel(dev.grads(), g) <= kTol, "train_step gradient", fmt(rel(dev.grads(), g)));
    report(rel(dev.rms_state(), v) <= 3 * kTol, "train_step RMS state", fmt(rel(dev.rms_state(), v)));

    // the pipelined form (submit_step / wait_step, two steps in flight) reproduces two
    // synchronous steps bit for bit
    const auto r2 = lamm_b200::train_step(dev, std::span<const lamm::Sample>(samples),
                                          std::span<const uint8_t>(denoise), tcfg, step + 1, 1, 0);
    lamm_b200::Device dev2(cfg, 0);
    dev2.set_params_from(params0);
    dev2.set_rms_state(std::vector<double>(g.size(), 0.0));
    dev2.set_reference_table(table);
    const int64_t t0 = lamm_b200::submit_step(dev2, std::span<const lamm::Sample>(samples),
                                              std::span<const uint8_t>(denoise), tcfg, step, 1, 0);
    const int64_t t1 = lamm_b200::submit_step(dev2, std::span<const lamm::Sample>(samples),
                                              std::span<const uint8_t>(denoise), tcfg, step + 1, 1, 0);
    const auto p0 = lamm_b200::wait_step(dev2, t0);
    const auto p1 = lamm_b200::wait_step(dev2, t1);
    report(p0.loss == r.loss && p1.loss == r2.loss && dev2.params() == dev.params(),
           "submit_step/wait_step == two train_step calls", fmt(std::abs(p1.loss - r2.loss)));
}

void check_evaluate(const std::vector<lamm::Sample>& samples, const lamm::model::ModelConfig& cfg,
                    const lamm::model::ModelParams& params, const lamm::loss::ReferenceTable& table) {
    const auto ref = lamm::trainer::evaluate(cfg, params, table, samples);
    lamm_b200::Device dev(cfg, 0);
    const auto got = lamm_b200::evaluate<lamm::trainer::EvalResult>(dev, cfg, params, table,
                                                                    std::span<const lamm::Sample>(samples));
    const double re = std::abs(got.energy_mae - ref.energy_mae) / std::abs(ref.energy_mae);
    const double rf = std::abs(got.force_mae - ref.force_mae) / std::abs(ref.force_mae);
    report(re <= kTol && rf <= kTol && got.energy_count == ref.energy_count && got.force_count == ref.force_count,
           "trainer::evaluate MAEs and counts", fmt(std::max(re, rf)));
}

void check_checkpoint(const lamm::model::ModelConfig& cfg, const lamm::model::ModelParams& params) {
    const std::string ours = "/tmp/lamm_b200_dropin_ours.ckpt", theirs = "/tmp/lamm_b200_dropin_ref.ckpt";
    lamm_b200::save_checkpoint(ours, cfg, params);
    lamm::model::save_checkpoint(theirs, cfg, params);
    const auto ref = lamm::model::load_checkpoint(ours);  // the reference reads ours
    auto mine = lamm::model::zero_like(params);
    const auto c = lamm_b200::load_checkpoint<lamm::model::ModelConfig>(theirs, mine);  // ours reads theirs
    report(ref.params == params && mine == params && c.hidden == cfg.hidden && c.heads == cfg.heads &&
               c.cutoff == cfg.cutoff,
           "LAMMCKPT save/load both ways, bit-exact");
}

}  // namespace

// PackedBatch::add_system keeps the cell of the FIRST system too (a one-sample
// periodic batch), zero rows for systems without one; the device then applies the
// minimum image: two atoms 9.5 A apart along x in a 10 A cubic cell are 0.5 A
// apart periodically (2 directed pairs), none without the cell.
void check_periodic_pack(lamm_b200::Device& dev, const lamm::model::ModelConfig& cfg) {
    lamm::AtomicSystem sys;
    sys.positions = {{0.25, 0.0, 0.0}, {9.75, 0.0, 0.0}};
    sys.atomic_numbers = {6, 8};
    const double cell[9] = {10.5, 0, 0, 0, 10.5, 0, 0, 0, 10.5};
    lamm_b200::PackedBatch one;
    one.add_system(sys, cell);
    const lamm_batch_view v = one.view();
    bool ok = v.cell != nullptr && one.cell.size() == 9 && one.cell[0] == 10.5 && one.cell[8] == 10.5;
    lamm_b200::PackedBatch two;
    two.add_system(sys);
    two.add_system(sys, cell);
    ok = ok && two.cell.size() == 18 && two.cell[0] == 0.0 && two.cell[9] == 10.5 && two.view().cell != nullptr;
    lamm_b200::PackedBatch none;
    none.add_system(sys);
    ok = ok && none.view().cell == nullptr;
    dev.set_batch(two);
    int64_t npairs = 0;
    lamm_b200::check(lamm_neighbor_list(dev.get(), &npairs));
    std::vector<int64_t> ptr(3);
    lamm_b200::check(lamm_neighbor_list_copy(dev.get(), ptr.data(), nullptr, nullptr, nullptr, nullptr));
    ok = ok && npairs == 2 && ptr[1] - ptr[0] == 0 && ptr[2] - ptr[1] == 2;
    report(ok, "PackedBatch: first system's cell kept, periodic pairs under the minimum image");
}

int main() {
    try {
        const lamm::model::ModelConfig cfg{128, 3, 16, 5.0, 4};
        const auto params = lamm::model::init_params(cfg, 7);
        auto mine = lamm::model::zero_like(params);
        lamm_b200::init_params(mine, cfg, 7);
        report(mine == params, "init_params bit-exact");
        const auto samples = make_samples(24, cfg.heads, 42);
        const auto table = make_table(cfg.heads);
        lamm_b200::Device dev(cfg, 0);
        check_neighbor_lists(dev, samples, cfg.cutoff);
        check_model(dev, samples, cfg, params, table);
        check_scheduler();
        check_train_step(samples, cfg, params, table);
        check_evaluate(samples, cfg, params, table);
        check_checkpoint(cfg, params);
        check_periodic_pack(dev, cfg);
        bool threw = false;
        try {
            lamm::model::ModelConfig bad = cfg;
            bad.hidden = 96;
            lamm_b200::Device d2(bad, 0);
        } catch (const lamm_b200::InputError&) {
            threw = true;
        }
        report(threw, "unsupported config -> InputError");
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d failure(s)\n", g_failures);
    return g_failures == 0 ? 0 : 1;
}
