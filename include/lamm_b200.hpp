// lamm_b200.hpp - C++ host layer over the C ABI (lamm_b200.h), shaped like the
// reference's lamm::core API so the hot path drops in with the reference's own
// types.
//
// Every entry point is a template over the caller's value types and only uses
// the members the reference declares, so `lamm::AtomicSystem`, `lamm::Sample`,
// `lamm::model::ModelParams`, `lamm::model::Prediction`, `lamm::NeighborList`,
// `lamm::scheduler::ScheduleConfig` / `MiniBatchSchedule` ... flow through
// unchanged (tests/cpp/test_dropin.cpp compiles it against the reference
// headers). Mapping (H = proj/core/include/lamm, S = proj/core/src):
//
//   lamm::build_neighbor_list          H/core.hpp:83          -> build_neighbor_list(dev, system, cutoff)
//   lamm::model::forward               H/model.hpp:123-124    -> forward(dev, system, params, cfg, cache*)
//   lamm::model::backward              H/model.hpp:128-129    -> backward(dev, cache, params, cfg, upstream, grads)
//   lamm::loss::masked_loss_grad       H/loss.hpp:81-84       -> masked_loss_grad(dev, cache, cfg, grads_out)
//   lamm::loss::normalize_labels       H/loss.hpp:58          -> Device::set_reference_table (applied on device)
//   lamm::scheduler::greedy_assign     H/scheduler.hpp:66-67  -> greedy_assign(atoms, G, B)
//   lamm::scheduler::plan              H/scheduler.hpp:74     -> plan<Schedule>(atoms, cfg)
//   lamm::model::init_params           H/model.hpp:75         -> init_params(params&, cfg, seed)
//   run_loop step body (file-local)    S/trainer.cpp:258-327  -> train_step(dev, samples, denoise, cfg, step, G, rank)
//                                                                train_step_workers(dev, samples, denoise, cfg, step, G)
//   lamm::trainer::evaluate            H/trainer.hpp:143-144  -> evaluate<EvalResult>(dev, cfg, params, refs, samples)
//   lamm::model::save/load_checkpoint  H/model.hpp:131-139    -> save_checkpoint(path, cfg, params), load_checkpoint
//
// Batched variants (forward_batch, build_neighbor_lists) take a span of
// systems and run them as one device-batch; the per-sample forms are the
// reference signatures with the Device prepended.
//
// Errors follow the reference: LAMM_EINPUT -> InputError (H/core.hpp:22-26),
// LAMM_ENONFINITE -> std::runtime_error (S/trainer.cpp:322-324), anything else
// -> DeviceError (a std::runtime_error). There is no CPU path: a missing GPU
// or library is an exception from the Device constructor.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lamm_b200.h"

namespace lamm_b200 {

struct InputError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NonFiniteError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int status) {
    if (status == LAMM_OK) return;
    const std::string msg = lamm_last_error();
    if (status == LAMM_EINPUT) throw InputError(msg);
    if (status == LAMM_ENONFINITE) throw NonFiniteError(msg);
    throw DeviceError(msg);
}

// ------------------------------------------------------------ configuration --
template <class ModelConfig>
lamm_model_config to_c(const ModelConfig& cfg) {
    lamm_model_config c{};
    c.hidden = cfg.hidden;
    c.layers = cfg.layers;
    c.rbf = cfg.rbf;
    c.heads = cfg.heads;
    c.cutoff = cfg.cutoff;
    return c;
}

// Step-body subset of lamm::trainer::TrainConfig (H/trainer.hpp:33-50).
// noise_scheme: anything whose integer value is 1 for "centered"
// (denoise::Scheme{baseline, centered}, H/denoise.hpp:19).
template <class TrainConfig>
lamm_train_config train_config_to_c(const TrainConfig& t) {
    lamm_train_config c{};
    c.learning_rate = t.learning_rate;
    c.clip_norm = t.clip_norm;
    c.rms_decay = t.rms_decay;
    c.rms_epsilon = t.rms_epsilon;
    c.noise_sigma = t.noise_sigma;
    c.noise_scheme = static_cast<int32_t>(t.noise_scheme);
    c.seed = t.seed;
    c.lambda_energy = t.lambda_energy;
    c.lambda_force = t.lambda_force;
    return c;
}

// ------------------------------------------------------------- parameters ----
// for_each_tensor order (H/model.hpp:59-66): embedding, filter[L], update[L],
// energy_head, force_head; each row-major rows() x cols() with data().
template <class Params, class F>
void for_each_tensor(Params& p, F&& fn) {
    fn(p.embedding);
    for (auto& m : p.filter) fn(m);
    for (auto& m : p.update) fn(m);
    fn(p.energy_head);
    fn(p.force_head);
}

template <class Params>
std::vector<double> flatten(const Params& p) {
    std::vector<double> out;
    lamm_b200::for_each_tensor(p, [&](const auto& m) { out.insert(out.end(), m.data(), m.data() + m.rows() * m.cols()); });
    return out;
}

template <class Params>
void unflatten(const std::vector<double>& flat, Params& p) {
    size_t off = 0;
    lamm_b200::for_each_tensor(p, [&](auto& m) {
        const size_t n = m.rows() * m.cols();
        if (off + n > flat.size()) throw InputError("unflatten: parameter vector too short");
        std::memcpy(m.data(), flat.data() + off, n * sizeof(double));
        off += n;
    });
    if (off != flat.size()) throw InputError("unflatten: parameter vector size mismatch");
}

// lamm::model::init_params (S/model.cpp:177-193) into caller-shaped params
// (the shapes of `params` must already match cfg, e.g. a zero_like copy).
template <class Params, class ModelConfig>
void init_params(Params& params, const ModelConfig& cfg, uint64_t seed) {
    const lamm_model_config c = to_c(cfg);
    std::vector<double> flat(static_cast<size_t>(lamm_param_count(&c)));
    check(lamm_init_params(&c, seed, flat.data()));
    unflatten(flat, params);
}

// --------------------------------------------------------------- batches -----
// Owning CSR pack of a device-batch (the lamm_batch_view layout).
struct PackedBatch {
    std::vector<int64_t> atom_ptr{0};
    std::vector<double> positions, energy, forces;
    std::vector<int32_t> Z, dataset_index;
    std::vector<uint8_t> energy_mask, force_mask, denoise;
    std::vector<double> cell;  // [B][9] periodic cells, empty if none was given (extension; see lamm_b200.h)
    std::vector<uint8_t> pbc;  // [B][3] per-axis periodicity of the cells (1 on all axes unless given)
    bool has_cell = false;     // some system carried a cell (then cell holds a row per system)

    int32_t size() const { return static_cast<int32_t>(atom_ptr.size() - 1); }
    int64_t atoms() const { return atom_ptr.back(); }

    // cell9: optional periodic cell of this system (rows = lattice vectors); pbc3:
    // optional per-axis periodicity of that cell (nullptr: periodic on all three
    // axes, e.g. {1, 1, 0} for a slab); the reference's AtomicSystem has neither
    template <class System>
    void add_system(const System& s, const double* cell9 = nullptr, const uint8_t* pbc3 = nullptr) {
        // once any system has a cell, every system has a [9] row (all zero:
        // non-periodic); the rows of the systems added before it are zero-filled
        if (cell9 != nullptr && !has_cell) {
            cell.assign(9 * static_cast<size_t>(size()), 0.0);
            pbc.assign(3 * static_cast<size_t>(size()), 1);
            has_cell = true;
        }
        if (has_cell) {
            for (int k = 0; k < 9; ++k) cell.push_back(cell9 ? cell9[k] : 0.0);
            for (int k = 0; k < 3; ++k) pbc.push_back(pbc3 ? (pbc3[k] ? 1 : 0) : 1);
        }
        const size_t n = s.positions.size();
        if (s.atomic_numbers.size() != n) throw InputError("system: positions / atomic_numbers size mismatch");
        for (size_t i = 0; i < n; ++i) {
            for (int c = 0; c < 3; ++c) positions.push_back(s.positions[i][c]);
            Z.push_back(static_cast<int32_t>(s.atomic_numbers[i]));
            for (int c = 0; c < 3; ++c) forces.push_back(0.0);
        }
        atom_ptr.push_back(atom_ptr.back() + static_cast<int64_t>(n));
        dataset_index.push_back(0);
        energy_mask.push_back(0);
        force_mask.push_back(0);
        energy.push_back(0.0);
        denoise.push_back(0);
    }

    // Sample = {system, labels{energy?, forces, energy_mask, force_mask,
    // dataset_index}} (H/core.hpp:50-65). `is_denoise` marks a sample of a
    // denoising subset: its labels come from make_denoising_sample on the device.
    template <class Sample>
    void add_sample(const Sample& s, bool is_denoise = false) {
        add_system(s.system);
        const size_t b = energy.size() - 1, n = s.system.positions.size();
        const auto& l = s.labels;
        dataset_index[b] = l.dataset_index;
        energy_mask[b] = l.energy_mask ? 1 : 0;
        force_mask[b] = l.force_mask ? 1 : 0;
        energy[b] = l.energy ? *l.energy : 0.0;
        if (!l.forces.empty()) {
            if (l.forces.size() != n) throw InputError("labels: forces rows != atoms");
            double* f = forces.data() + 3 * (atom_ptr[b]);
            for (size_t i = 0; i < n; ++i)
                for (int c = 0; c < 3; ++c) f[3 * i + c] = l.forces[i][c];
        }
        denoise[b] = is_denoise ? 1 : 0;
    }

    lamm_batch_view view() const {
        lamm_batch_view v{};
        v.n_samples = size();
        v.n_atoms = atoms();
        v.atom_ptr = atom_ptr.data();
        v.positions = positions.data();
        v.atomic_numbers = Z.data();
        v.dataset_index = dataset_index.data();
        v.energy_mask = energy_mask.data();
        v.force_mask = force_mask.data();
        v.energy = energy.data();
        v.forces = forces.data();
        v.denoise = denoise.data();
        v.cell = has_cell ? cell.data() : nullptr;
        v.pbc = has_cell ? pbc.data() : nullptr;
        return v;
    }
};

// ----------------------------------------------------------------- device ----
// One lamm_ctx: one GPU, one stream, one host thread (H/core.hpp threading
// note: reentrant on const inputs; a Device is not).
class Device {
public:
    template <class ModelConfig>
    explicit Device(const ModelConfig& cfg, int device = 0) : cfg_(to_c(cfg)) {
        lamm_ctx* c = nullptr;
        check(lamm_ctx_create(device, &cfg_, &c));
        ctx_.reset(c);
        n_params_ = static_cast<size_t>(lamm_param_count(&cfg_));
    }
    lamm_ctx* get() const { return ctx_.get(); }
    const lamm_model_config& config() const { return cfg_; }
    size_t param_count() const { return n_params_; }

    void set_option(const char* name, int64_t v) { check(lamm_ctx_set_option(get(), name, v)); }

    // Parameters are uploaded only when they differ from the resident copy.
    void set_params(const std::vector<double>& flat) {
        if (flat.size() != n_params_) throw InputError("params: size does not match the model config");
        if (flat == resident_) return;
        check(lamm_params_set(get(), flat.data(), flat.size()));
        resident_ = flat;
    }
    template <class Params>
    void set_params_from(const Params& p) {
        set_params(flatten(p));
    }
    std::vector<double> params() const {
        std::vector<double> out(n_params_);
        check(lamm_params_get(get(), out.data(), out.size()));
        return out;
    }
    void params_changed_on_device() { resident_.clear(); }
    // RMS optimizer state v (S/trainer.cpp:29-35), for_each_tensor layout.
    void set_rms_state(const std::vector<double>& v) {
        if (v.size() != n_params_) throw InputError("rms state: size does not match the model config");
        check(lamm_rms_state_set(get(), v.data(), v.size()));
    }
    std::vector<double> rms_state() const {
        std::vector<double> out(n_params_);
        check(lamm_rms_state_get(get(), out.data(), out.size()));
        return out;
    }
    // Gradient of the last train step (sum over workers, before /G).
    std::vector<double> grads() const {
        std::vector<double> out(n_params_);
        check(lamm_grads_get(get(), out.data(), out.size()));
        return out;
    }

    // ReferenceTable {per_dataset[d]: DatasetNormalizer} (H/loss.hpp:31-44);
    // normalize_labels (S/loss.cpp:113-126) then runs on the device.
    template <class ReferenceTable>
    void set_reference_table(const ReferenceTable& t) {
        const size_t D = t.per_dataset.size();
        std::vector<double> rho(D * 119, 0.0), mean(D), std_(D), fstd(D);
        std::vector<uint8_t> rho_has(D * 119, 0), has(D);
        for (size_t d = 0; d < D; ++d) {
            const auto& n = t.per_dataset[d];
            for (const auto& [z, v] : n.reference_energies) {
                if (z < 1 || z > 118) throw InputError("reference table: Z out of range");
                rho[d * 119 + z] = v;
                rho_has[d * 119 + z] = 1;
            }
            mean[d] = n.energy_mean;
            std_[d] = n.energy_std;
            fstd[d] = n.force_std;
            has[d] = n.has_energy_stats ? 1 : 0;
        }
        lamm_ref_table c{static_cast<int32_t>(D), rho.data(), rho_has.data(), mean.data(), std_.data(), fstd.data(),
                         has.data()};
        check(lamm_ref_table_set(get(), &c));
    }
    void clear_reference_table() { check(lamm_ref_table_set(get(), nullptr)); }

    void set_batch(const PackedBatch& b) {
        const lamm_batch_view v = b.view();
        check(lamm_batch_set(get(), &v));
        batch_atom_ptr_ = b.atom_ptr;
        ++generation_;
    }
    const std::vector<int64_t>& batch_atom_ptr() const { return batch_atom_ptr_; }
    void batch_replaced(const std::vector<int64_t>& atom_ptr) {  // a call uploaded its own batch
        batch_atom_ptr_ = atom_ptr;
        ++generation_;
    }
    uint64_t generation() const { return generation_; }

    void comm_init(int nranks, int rank, const void* unique_id128) {
        check(lamm_comm_init(get(), nranks, rank, unique_id128));
    }
    static std::array<unsigned char, 128> comm_unique_id() {
        std::array<unsigned char, 128> id{};
        check(lamm_comm_unique_id(id.data()));
        return id;
    }
    void sync() { check(lamm_sync(get())); }

private:
    struct Del {
        void operator()(lamm_ctx* c) const { lamm_ctx_destroy(c); }
    };
    lamm_model_config cfg_{};
    std::unique_ptr<lamm_ctx, Del> ctx_;
    size_t n_params_ = 0;
    std::vector<double> resident_;
    std::vector<int64_t> batch_atom_ptr_;
    uint64_t generation_ = 0;
};

// Device-side stand-in for lamm::model::ForwardCache (H/model.hpp:79-88): the
// intermediates stay in HBM; this handle names the device-batch they belong to.
struct DeviceCache {
    const Device* device = nullptr;
    uint64_t generation = 0;
    std::vector<int64_t> atom_ptr;

    void require_current(const Device& dev) const {
        if (device != &dev || generation != dev.generation())
            throw InputError("forward cache is stale: the device ran another batch since this forward");
    }
};

// ------------------------------------------------------- neighbour lists -----
// lamm::build_neighbor_list (H/core.hpp:83, S/core.cpp:30-48) for every system
// of a device-batch: bit-exact pair set, order, distance and unit.
template <class NeighborList, class System>
std::vector<NeighborList> build_neighbor_lists(Device& dev, std::span<const System> systems, double cutoff) {
    if (!(cutoff == dev.config().cutoff))
        throw InputError("build_neighbor_list: the device model was created for another cutoff");
    PackedBatch b;
    for (const auto& s : systems) b.add_system(s);
    dev.set_batch(b);
    dev.set_option("export_fp64", 1);
    int64_t P = 0;
    check(lamm_neighbor_list(dev.get(), &P));
    std::vector<int64_t> ptr(systems.size() + 1);
    std::vector<int32_t> pi(P), pj(P);
    std::vector<double> dist(P), unit(3 * P);
    check(lamm_neighbor_list_copy(dev.get(), ptr.data(), pi.data(), pj.data(), dist.data(), unit.data()));
    dev.set_option("export_fp64", 0);
    std::vector<NeighborList> out(systems.size());
    for (size_t s = 0; s < systems.size(); ++s) {
        out[s].cutoff = cutoff;
        out[s].pairs.resize(static_cast<size_t>(ptr[s + 1] - ptr[s]));
        for (int64_t p = ptr[s]; p < ptr[s + 1]; ++p) {
            auto& q = out[s].pairs[static_cast<size_t>(p - ptr[s])];
            q.i = pi[p];
            q.j = pj[p];
            q.distance = dist[p];
            q.unit = {unit[3 * p], unit[3 * p + 1], unit[3 * p + 2]};
        }
    }
    return out;
}

template <class NeighborList, class System>
NeighborList build_neighbor_list(Device& dev, const System& system, double cutoff) {
    return build_neighbor_lists<NeighborList, System>(dev, std::span<const System>(&system, 1), cutoff)[0];
}

// ----------------------------------------------------------------- model -----
// lamm::model::forward (H/model.hpp:123-124) for a device-batch: Prediction
// {n_atoms, heads, energy[D], forces[D*N*3] at (d*N+j)*3+c} per system.
template <class Prediction, class System, class Params, class ModelConfig>
std::vector<Prediction> forward_batch(Device& dev, std::span<const System> systems, const Params& params,
                                      const ModelConfig& cfg, DeviceCache* cache = nullptr) {
    const lamm_model_config c = to_c(cfg);
    if (std::memcmp(&c, &dev.config(), sizeof c) != 0) throw InputError("forward: model config differs from the device's");
    dev.set_params_from(params);
    PackedBatch b;
    for (const auto& s : systems) b.add_system(s);
    dev.set_batch(b);
    const int D = c.heads;
    std::vector<double> e(static_cast<size_t>(b.size()) * D), f(static_cast<size_t>(b.atoms()) * 3 * D);
    check(lamm_forward(dev.get(), e.data(), f.data()));
    std::vector<Prediction> out(systems.size());
    for (size_t s = 0; s < systems.size(); ++s) {
        const int64_t a0 = b.atom_ptr[s], n = b.atom_ptr[s + 1] - a0;
        out[s].n_atoms = static_cast<int>(n);
        out[s].heads = D;
        out[s].energy.assign(e.begin() + s * D, e.begin() + (s + 1) * D);
        out[s].forces.assign(f.begin() + 3 * D * a0, f.begin() + 3 * D * (a0 + n));
    }
    if (cache) *cache = DeviceCache{&dev, dev.generation(), b.atom_ptr};
    return out;
}

template <class Prediction, class System, class Params, class ModelConfig>
Prediction forward(Device& dev, const System& system, const Params& params, const ModelConfig& cfg,
                   DeviceCache* cache = nullptr) {
    return forward_batch<Prediction>(dev, std::span<const System>(&system, 1), params, cfg, cache)[0];
}

// lamm::model::backward (H/model.hpp:128-129, S/model.cpp:299-425) for the
// device-batch of `cache`, upstream per system in Prediction layout;
// accumulates (+=) into grads like the reference.
template <class Params, class ModelConfig, class PredictionGrad, class Gradients>
void backward(Device& dev, const DeviceCache& cache, const Params& params, const ModelConfig& cfg,
              std::span<const PredictionGrad> upstream, Gradients& grads) {
    cache.require_current(dev);
    (void)cfg;
    dev.set_params_from(params);
    const int D = dev.config().heads;
    const size_t B = cache.atom_ptr.size() - 1;
    if (upstream.size() != B) throw InputError("backward: one upstream gradient per system of the cached batch");
    std::vector<double> ge(B * D), gf(static_cast<size_t>(cache.atom_ptr.back()) * 3 * D);
    for (size_t s = 0; s < B; ++s) {
        const int64_t a0 = cache.atom_ptr[s], n = cache.atom_ptr[s + 1] - a0;
        if (upstream[s].energy.size() != static_cast<size_t>(D) ||
            upstream[s].forces.size() != static_cast<size_t>(3 * D * n))
            throw InputError("backward: upstream gradient shape does not match the prediction");
        std::copy(upstream[s].energy.begin(), upstream[s].energy.end(), ge.begin() + s * D);
        std::copy(upstream[s].forces.begin(), upstream[s].forces.end(), gf.begin() + 3 * D * a0);
    }
    std::vector<double> acc = flatten(grads);
    check(lamm_backward(dev.get(), ge.data(), gf.data(), acc.data()));
    unflatten(acc, grads);
}

// ------------------------------------------------------------------ loss -----
// lamm::loss::masked_loss_grad (H/loss.hpp:81-84, S/loss.cpp:140-226) on the
// predictions of the cached forward and the labels of its batch (set with
// Device::set_batch from samples). grads_out gets one PredictionGrad per sample.
template <class LossBreakdown, class LossConfig, class PredictionGrad>
LossBreakdown masked_loss_grad(Device& dev, const DeviceCache& cache, const LossConfig& cfg,
                               std::vector<PredictionGrad>& grads_out) {
    cache.require_current(dev);
    const lamm_loss_config c{cfg.lambda_energy, cfg.lambda_force};
    const int D = dev.config().heads;
    const size_t B = cache.atom_ptr.size() - 1;
    std::vector<double> ge(B * D), gf(static_cast<size_t>(cache.atom_ptr.back()) * 3 * D);
    lamm_loss_breakdown lb{};
    check(lamm_loss_grad(dev.get(), &c, &lb, ge.data(), gf.data()));
    grads_out.resize(B);
    for (size_t s = 0; s < B; ++s) {
        const int64_t a0 = cache.atom_ptr[s], n = cache.atom_ptr[s + 1] - a0;
        grads_out[s].n_atoms = static_cast<int>(n);
        grads_out[s].heads = D;
        grads_out[s].energy.assign(ge.begin() + s * D, ge.begin() + (s + 1) * D);
        grads_out[s].forces.assign(gf.begin() + 3 * D * a0, gf.begin() + 3 * D * (a0 + n));
    }
    LossBreakdown out{};
    out.total = lb.total;
    out.energy_term = lb.energy_term;
    out.force_term = lb.force_term;
    out.energy_labeled = lb.energy_labeled;
    out.force_labeled = lb.force_labeled;
    out.energy_empty = lb.energy_empty != 0;
    out.force_empty = lb.force_empty != 0;
    return out;
}

// Forward of labelled samples: packs labels with the systems so that
// masked_loss_grad can run on the device afterwards.
template <class Prediction, class Sample, class Params, class ModelConfig>
std::vector<Prediction> forward_samples(Device& dev, std::span<const Sample> samples, const Params& params,
                                        const ModelConfig& cfg, DeviceCache* cache) {
    const lamm_model_config c = to_c(cfg);
    if (std::memcmp(&c, &dev.config(), sizeof c) != 0) throw InputError("forward: model config differs from the device's");
    dev.set_params_from(params);
    PackedBatch b;
    for (const auto& s : samples) b.add_sample(s);
    dev.set_batch(b);
    const int D = c.heads;
    std::vector<double> e(static_cast<size_t>(b.size()) * D), f(static_cast<size_t>(b.atoms()) * 3 * D);
    check(lamm_forward(dev.get(), e.data(), f.data()));
    std::vector<Prediction> out(samples.size());
    for (size_t s = 0; s < samples.size(); ++s) {
        const int64_t a0 = b.atom_ptr[s], n = b.atom_ptr[s + 1] - a0;
        out[s].n_atoms = static_cast<int>(n);
        out[s].heads = D;
        out[s].energy.assign(e.begin() + s * D, e.begin() + (s + 1) * D);
        out[s].forces.assign(f.begin() + 3 * D * a0, f.begin() + 3 * D * (a0 + n));
    }
    if (cache) *cache = DeviceCache{&dev, dev.generation(), b.atom_ptr};
    return out;
}

// ------------------------------------------------------------ train step -----
struct StepResult {
    double loss = 0.0;       // mean over workers of the per-worker Eq.(5) loss (S/trainer.cpp:320)
    double grad_norm = 0.0;  // before clipping (S/trainer.cpp:321)
    lamm_loss_breakdown local{};
    int64_t atoms = 0, edges = 0;
};

// One optimizer step with the semantics of S/trainer.cpp:258-327 for worker
// `rank` of `workers`: `samples` are MiniBatch.samples[rank*B .. rank*B+B)
// resolved to Samples (raw labels; the device normalizes with the table set on
// `dev`), denoise[b] marks samples of denoising subsets. Parameters and the RMS
// state stay on the device; read them with Device::params().
template <class Sample, class TrainConfig>
StepResult train_step(Device& dev, std::span<const Sample> samples, std::span<const uint8_t> denoise,
                      const TrainConfig& tcfg, int64_t step, int workers = 1, int rank = 0) {
    if (!denoise.empty() && denoise.size() != samples.size())
        throw InputError("train_step: one denoise flag per sample");
    PackedBatch b;
    for (size_t s = 0; s < samples.size(); ++s) b.add_sample(samples[s], !denoise.empty() && denoise[s] != 0);
    const lamm_batch_view v = b.view();
    const lamm_train_config c = train_config_to_c(tcfg);
    lamm_step_result r{};
    const int st = lamm_train_step(dev.get(), &v, &c, step, workers, rank, &r);
    dev.params_changed_on_device();
    dev.batch_replaced(b.atom_ptr);  // earlier DeviceCaches are stale now
    check(st);
    return StepResult{r.loss, r.grad_norm, r.local, r.n_atoms, r.n_edges};
}

// Pipelined form of train_step (lamm_train_step_submit / lamm_train_step_wait):
// submit_step packs and enqueues the step and returns its ticket without waiting,
// so the host can pack step k+1 while the device runs step k; wait_step returns
// the oldest outstanding step's result. At most two in flight, waited in order;
// the results and parameters equal the synchronous sequence.
template <class Sample, class TrainConfig>
int64_t submit_step(Device& dev, std::span<const Sample> samples, std::span<const uint8_t> denoise,
                    const TrainConfig& tcfg, int64_t step, int workers = 1, int rank = 0) {
    if (!denoise.empty() && denoise.size() != samples.size())
        throw InputError("submit_step: one denoise flag per sample");
    PackedBatch b;
    for (size_t s = 0; s < samples.size(); ++s) b.add_sample(samples[s], !denoise.empty() && denoise[s] != 0);
    const lamm_batch_view v = b.view();
    const lamm_train_config c = train_config_to_c(tcfg);
    int64_t ticket = -1;
    const int st = lamm_train_step_submit(dev.get(), &v, &c, step, workers, rank, &ticket);  // packed: b may go
    dev.batch_replaced(b.atom_ptr);  // the device batch is this step's from now on
    check(st);
    return ticket;
}

inline StepResult wait_step(Device& dev, int64_t ticket) {
    lamm_step_result r{};
    const int st = lamm_train_step_wait(dev.get(), ticket, &r);
    dev.params_changed_on_device();
    check(st);
    return StepResult{r.loss, r.grad_norm, r.local, r.n_atoms, r.n_edges};
}

// The step of S/trainer.cpp:258-327 for all G workers SIMULATED on this one
// device, in worker order: `samples` is the whole MiniBatch (G*B, worker-major),
// denoise[k] marks samples of denoising subsets (empty: none).
template <class Sample, class TrainConfig>
StepResult train_step_workers(Device& dev, std::span<const Sample> samples, std::span<const uint8_t> denoise,
                              const TrainConfig& tcfg, int64_t step, int workers) {
    if (workers < 1 || samples.size() % static_cast<size_t>(workers) != 0)
        throw InputError("train_step_workers: samples must split into `workers` equal device-batches");
    if (!denoise.empty() && denoise.size() != samples.size())
        throw InputError("train_step_workers: one denoise flag per sample");
    const size_t B = samples.size() / static_cast<size_t>(workers);
    std::vector<PackedBatch> packs(static_cast<size_t>(workers));
    std::vector<lamm_batch_view> views;
    for (int g = 0; g < workers; ++g) {
        for (size_t b = 0; b < B; ++b) {
            const size_t k = static_cast<size_t>(g) * B + b;
            packs[static_cast<size_t>(g)].add_sample(samples[k], !denoise.empty() && denoise[k] != 0);
        }
    }
    for (auto& p : packs) views.push_back(p.view());
    const lamm_train_config c = train_config_to_c(tcfg);
    lamm_step_result r{};
    const int st = lamm_train_step_workers(dev.get(), views.data(), workers, &c, step, &r);
    dev.params_changed_on_device();
    if (st == LAMM_OK || st == LAMM_ENONFINITE) dev.batch_replaced(packs.back().atom_ptr);
    check(st);
    return StepResult{r.loss, r.grad_norm, r.local, r.n_atoms, r.n_edges};
}

// ------------------------------------------------------------ evaluation -----
// lamm::trainer::evaluate (H/trainer.hpp:143-144, S/trainer.cpp:528-553):
// EvalResult {energy_mae, force_mae, energy_count, force_count} of the device's
// parameters on `samples` (raw labels), denormalized with its reference table.
template <class EvalResult, class Sample>
EvalResult evaluate(Device& dev, std::span<const Sample> samples) {
    PackedBatch b;
    for (const auto& s : samples) b.add_sample(s);
    const lamm_batch_view v = b.view();
    lamm_eval_result r{};
    check(lamm_evaluate(dev.get(), &v, &r));
    dev.batch_replaced(b.atom_ptr);
    EvalResult out{};
    out.energy_mae = r.energy_mae;
    out.force_mae = r.force_mae;
    out.energy_count = r.energy_count;
    out.force_count = r.force_count;
    return out;
}

// The reference signature: parameters and table installed first.
template <class EvalResult, class ModelConfig, class Params, class ReferenceTable, class Sample>
EvalResult evaluate(Device& dev, const ModelConfig& cfg, const Params& params, const ReferenceTable& refs,
                    std::span<const Sample> samples) {
    const lamm_model_config c = to_c(cfg);
    if (std::memcmp(&c, &dev.config(), sizeof c) != 0) throw InputError("evaluate: model config differs from the device's");
    dev.set_params_from(params);
    dev.set_reference_table(refs);
    return evaluate<EvalResult>(dev, samples);
}

// ------------------------------------------------------------ checkpoints ----
// lamm::model::save_checkpoint / load_checkpoint (H/model.hpp:131-139): the same
// LAMMCKPT bytes. Checkpoint = {config, params} like the reference's struct; the
// params object must come shaped (e.g. init_params of the config, or the
// reference's own load) - unflatten checks the size.
template <class ModelConfig, class Params>
void save_checkpoint(const std::string& path, const ModelConfig& cfg, const Params& params) {
    const lamm_model_config c = to_c(cfg);
    const std::vector<double> flat = flatten(params);
    check(lamm_checkpoint_save(path.c_str(), &c, flat.data(), flat.size()));
}

// Reads a checkpoint into caller-shaped params; returns its config.
template <class ModelConfig, class Params>
ModelConfig load_checkpoint(const std::string& path, Params& params) {
    lamm_model_config c{};
    size_t n = 0;
    check(lamm_checkpoint_load(path.c_str(), &c, nullptr, 0, &n));
    std::vector<double> flat(n);
    check(lamm_checkpoint_load(path.c_str(), &c, flat.data(), flat.size(), &n));
    unflatten(flat, params);
    ModelConfig out{};
    out.hidden = c.hidden;
    out.layers = c.layers;
    out.rbf = c.rbf;
    out.heads = c.heads;
    out.cutoff = c.cutoff;
    return out;
}

// ------------------------------------------------------------- scheduler -----
// lamm::scheduler::greedy_assign (S/scheduler.cpp:62-89): worker per input.
inline std::vector<int> greedy_assign(const std::vector<int64_t>& atoms, int workers, int batch_per_worker) {
    std::vector<int32_t> w(atoms.size());
    check(lamm_greedy_assign(atoms.data(), static_cast<int64_t>(atoms.size()), workers, batch_per_worker, w.data()));
    return std::vector<int>(w.begin(), w.end());
}

// lamm::scheduler::plan (S/scheduler.cpp:91-203) into the caller's
// MiniBatchSchedule {batches[MiniBatch{samples[ScheduledSample], worker_atoms}],
// workers, batch_per_worker, dropped_samples}. cfg.mode: enum whose integer
// values are {balanced 0, greedy_only 1, naive 2} (H/scheduler.hpp:28).
template <class Schedule, class ScheduleConfig>
Schedule plan(const std::vector<int64_t>& atoms, const ScheduleConfig& cfg) {
    const int64_t n = static_cast<int64_t>(atoms.size());
    std::vector<int64_t> sample(n), a(n), split(n), rank(n), watoms(n + 1);
    std::vector<int32_t> worker(n);
    int64_t nb = 0, dropped = 0;
    check(lamm_plan(atoms.data(), n, cfg.workers, cfg.batch_per_worker, cfg.num_splits, cfg.seed,
                    static_cast<int32_t>(cfg.mode), sample.data(), worker.data(), a.data(), split.data(), rank.data(),
                    watoms.data(), &nb, &dropped));
    Schedule out{};
    out.workers = cfg.workers;
    out.batch_per_worker = cfg.batch_per_worker;
    out.dropped_samples = dropped;
    const int64_t per = static_cast<int64_t>(cfg.workers) * cfg.batch_per_worker;
    out.batches.resize(static_cast<size_t>(nb));
    for (int64_t s = 0; s < nb; ++s) {
        auto& mb = out.batches[static_cast<size_t>(s)];
        mb.samples.resize(static_cast<size_t>(per));
        for (int64_t k = 0; k < per; ++k) {
            auto& q = mb.samples[static_cast<size_t>(k)];
            const int64_t x = s * per + k;
            q.sample = sample[x];
            q.worker = worker[x];
            q.atoms = a[x];
            q.split = split[x];
            q.chunk_rank = rank[x];
        }
        mb.worker_atoms.assign(watoms.begin() + s * cfg.workers, watoms.begin() + (s + 1) * cfg.workers);
    }
    return out;
}

}  // namespace lamm_b200
