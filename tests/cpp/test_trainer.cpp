// test_trainer.cpp - orchestration parity:
// lamm_b200::trainer::{pretrain, finetune, denoise_bench}
// (include/lamm_b200_trainer.hpp, device step) against the reference's
// lamm::trainer::{pretrain, finetune, denoise_bench} (CPU, fp64) called in the
// same binary on the same synthetic catalog and seeds.
//
// Test infrastructure: built by oracle/Makefile (target `trainer`) from the
// reference sources under /root/reference into oracle/_ref/test_trainer, linked
// against the product library; run by tests/test_cxx_dropin.py on a GPU.
//
// Bars: the run structure is exact (metric points, their steps and splits,
// checkpoint-sink steps, reference tables, steps-to-threshold); losses, MAEs
// and final parameters within the 1e-4 step bar over the whole run (measured
// on B200: <= 5e-6 relative). A trajectory can in principle leave that bar: the
// RMS optimizer's first step moves a parameter by ~10 lr sign(g), so a gradient
// element that is ~0 in fp64 could take the other sign in fp32.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "lamm/dataset.hpp"
#include "lamm/model.hpp"
#include "lamm/scheduler.hpp"
#include "lamm/trainer.hpp"
#include "lamm_b200_trainer.hpp"

namespace {

int g_failures = 0;
constexpr double kLossTol = 1e-4;   // relative, per emitted train loss
constexpr double kMaeTol = 1e-4;    // relative, per emitted MAE
constexpr double kParamTol = 1e-4;  // ||p - p_ref|| / ||p_ref|| after the run

void report(bool ok, const std::string& what, const std::string& detail = "") {
    std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", what.c_str(), detail.empty() ? "" : "  ", detail.c_str());
    if (!ok) ++g_failures;
}

double rel1(double a, double b) {
    if (std::isnan(a) || std::isnan(b)) return std::isnan(a) && std::isnan(b) ? 0.0 : INFINITY;
    return std::abs(a - b) / std::max(std::abs(b), 1e-12);
}

std::vector<double> flat(const lamm::model::ModelParams& p) { return lamm_b200::flatten(p); }

double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
    double d2 = 0, r2 = 0;
    for (size_t k = 0; k < a.size(); ++k) d2 += (a[k] - b[k]) * (a[k] - b[k]), r2 += b[k] * b[k];
    return std::sqrt(d2 / r2);
}

void compare_metrics(const std::string& what, const lamm::trainer::RunMetrics& mine,
                     const lamm::trainer::RunMetrics& ref) {
    bool shape = mine.points.size() == ref.points.size();
    double worst_loss = 0, worst_mae = 0;
    for (size_t k = 0; shape && k < ref.points.size(); ++k) {
        const auto &a = mine.points[k], &b = ref.points[k];
        shape = shape && a.step == b.step && a.split == b.split;
        if (b.split == "train") worst_loss = std::max(worst_loss, rel1(a.loss, b.loss));
        worst_mae = std::max({worst_mae, rel1(a.energy_mae, b.energy_mae), rel1(a.force_mae, b.force_mae)});
    }
    report(shape, what + ": metric points (step, split) identical",
           std::to_string(mine.points.size()) + " points");
    char buf[160];
    std::snprintf(buf, sizeof buf, "max rel %.2e (tol %.0e)", worst_loss, kLossTol);
    report(worst_loss <= kLossTol, what + ": train losses", buf);
    std::snprintf(buf, sizeof buf, "max rel %.2e (tol %.0e)", worst_mae, kMaeTol);
    report(worst_mae <= kMaeTol, what + ": energy/force MAEs (train batch stats + val)", buf);
    std::snprintf(buf, sizeof buf, "%.3e vs %.3e", mine.final_loss, ref.final_loss);
    report(rel1(mine.final_loss, ref.final_loss) <= kLossTol, what + ": final loss", buf);
    report(rel1(mine.best_energy_mae, ref.best_energy_mae) <= kMaeTol &&
               rel1(mine.best_force_mae, ref.best_force_mae) <= kMaeTol,
           what + ": best val MAEs");
}

// The tables: the same elements, head flags and force std (bit for bit: the same
// fixed-order sums, and the pseudo-force probe's noise draws); the reference
// energies and residual statistics within 1e-9 relative - the library solves the
// minimum-norm least squares with its own complete orthogonal decomposition, the
// reference build here with oracle/shim's Eigen stand-in (parity-unpinned).
bool same_table(const lamm::loss::ReferenceTable& a, const lamm::loss::ReferenceTable& b) {
    if (a.per_dataset.size() != b.per_dataset.size()) return false;
    auto close = [](double u, double v) { return std::fabs(u - v) <= 1e-9 * std::max(1.0, std::fabs(v)); };
    for (size_t d = 0; d < a.per_dataset.size(); ++d) {
        const auto &x = a.per_dataset[d], &y = b.per_dataset[d];
        if (x.reference_energies.size() != y.reference_energies.size() || x.force_std != y.force_std ||
            x.has_energy_stats != y.has_energy_stats || !close(x.energy_mean, y.energy_mean) ||
            !close(x.energy_std, y.energy_std))
            return false;
        for (const auto& [z, v] : y.reference_energies) {
            const auto it = x.reference_energies.find(z);
            if (it == x.reference_energies.end() || !close(it->second, v)) return false;
        }
    }
    return true;
}

lamm::dataset::Catalog make_catalog() {
    std::vector<lamm::dataset::SynthSpec> specs(3);
    specs[0].name = "molecules";
    specs[0].count = 96;
    specs[0].atom_count_mode = 10.0;
    specs[0].max_atoms = 40;
    specs[0].elements = {1, 6, 8};
    specs[1].name = "energy_only";
    specs[1].task = lamm::dataset::TaskKind::energy_only;
    specs[1].count = 64;
    specs[1].atom_count_mode = 14.0;
    specs[1].max_atoms = 48;
    specs[1].elements = {6, 7};
    specs[2].name = "unlabeled";
    specs[2].task = lamm::dataset::TaskKind::denoising;
    specs[2].count = 48;
    specs[2].atom_count_mode = 12.0;
    specs[2].max_atoms = 40;
    specs[2].elements = {6, 8};
    return lamm::dataset::synth_catalog(specs, 2024);
}

}  // namespace

int main() {
    try {
        const auto catalog = make_catalog();
        const lamm::model::ModelConfig mcfg{32, 2, 8, 5.0, 3};
        lamm::scheduler::ScheduleConfig sched;
        sched.workers = 2;
        sched.batch_per_worker = 4;
        sched.num_splits = 8;
        lamm::trainer::TrainConfig tc;
        tc.max_steps = 8;
        tc.val_every = 3;
        tc.checkpoint_every = 4;
        tc.val_fraction = 0.1;
        tc.seed = 11;
        lamm::dataset::MixPlan mix;
        mix.temperature = 2.0;

        // ---- pretrain
        std::vector<int64_t> ref_ck, my_ck;
        const auto ref = lamm::trainer::pretrain(
            catalog, mix, sched, mcfg, tc,
            [&](int64_t s, const auto&, const auto&, const auto&) { ref_ck.push_back(s); });
        const auto mine = lamm_b200::trainer::pretrain(
            catalog, mix, sched, mcfg, tc,
            [&](int64_t s, const auto&, const auto&, const auto&) { my_ck.push_back(s); });
        report(same_table(mine.refs, ref.refs), "pretrain: reference tables (elements, flags, force std exact; rho/mean/std 1e-9)");
        report(my_ck == ref_ck, "pretrain: checkpoint-sink steps identical", std::to_string(my_ck.size()) + " calls");
        compare_metrics("pretrain", mine.metrics, ref.metrics);
        const double dp = rel_l2(flat(mine.params), flat(ref.params));
        char buf[128];
        std::snprintf(buf, sizeof buf, "||d||/||ref|| %.2e (tol %.0e)", dp, kParamTol);
        report(dp <= kParamTol, "pretrain: final parameters", buf);

        // ---- finetune from the reference's pretrained checkpoint, one fresh head
        lamm::model::Checkpoint start{ref.config, ref.params};
        lamm::trainer::TrainConfig ft = tc;
        ft.max_steps = 5;
        ft.val_every = 2;
        ft.checkpoint_every = 0;
        ft.val_fraction = 0.15;
        const auto ref_ft = lamm::trainer::finetune(start, catalog.subsets[0], sched, ft);
        const auto my_ft = lamm_b200::trainer::finetune(start, catalog.subsets[0], sched, ft);
        report(my_ft.config.heads == 1 && ref_ft.config.heads == 1, "finetune: single head");
        report(same_table(my_ft.refs, ref_ft.refs), "finetune: reference tables (elements, flags, force std exact; rho/mean/std 1e-9)");
        compare_metrics("finetune", my_ft.metrics, ref_ft.metrics);
        const double dft = rel_l2(flat(my_ft.params), flat(ref_ft.params));
        std::snprintf(buf, sizeof buf, "||d||/||ref|| %.2e (tol %.0e)", dft, kParamTol);
        report(dft <= kParamTol, "finetune: final parameters", buf);

        // ---- denoise_bench: baseline vs centered labels on the unlabeled subset
        lamm::trainer::TrainConfig db = tc;
        db.max_steps = 6;
        db.val_every = 2;
        db.val_fraction = 0.2;
        const auto ref_db = lamm::trainer::denoise_bench(catalog.subsets[2], sched, mcfg, db, 1e9);
        const auto my_db = lamm_b200::trainer::denoise_bench(catalog.subsets[2], sched, mcfg, db, 1e9);
        compare_metrics("denoise_bench baseline", my_db.baseline, ref_db.baseline);
        compare_metrics("denoise_bench centered", my_db.centered, ref_db.centered);
        report(my_db.baseline_steps_to_threshold == ref_db.baseline_steps_to_threshold &&
                   my_db.centered_steps_to_threshold == ref_db.centered_steps_to_threshold,
               "denoise_bench: steps to threshold identical",
               std::to_string(my_db.baseline_steps_to_threshold) + ", " +
                   std::to_string(my_db.centered_steps_to_threshold));

        // ---- errors follow the reference
        bool threw = false;
        try {
            lamm::trainer::TrainConfig bad = tc;
            bad.val_every = 0;
            lamm_b200::trainer::pretrain(catalog, mix, sched, mcfg, bad);
        } catch (const lamm::InputError&) {
            threw = true;
        }
        report(threw, "invalid TrainConfig -> InputError");
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d failure(s)\n", g_failures);
    return g_failures == 0 ? 0 : 1;
}
