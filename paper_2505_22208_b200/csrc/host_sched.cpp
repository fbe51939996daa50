// host_sched.cpp - LaMM's atom-count load balancer and the host-side data
// generators, written for the B200 path's host runtime (liblamm_b200.so).
//
// These run once per epoch (plan) or once per run (generators) on the host;
// the GPU path only consumes their output. Results are bit-exact with the
// reference (checked against oracle/_ref by tests/test_host_parity.py):
//   greedy_assign ...... S/scheduler.cpp:62-89   (LPT with a cap of B per worker)
//   plan_balanced ...... S/scheduler.cpp:91-158  (shuffle -> S sorted splits ->
//                                                  transpose chunk stream -> greedy)
//   plan_naive ......... S/scheduler.cpp:160-199
//   schedule_metrics ... S/scheduler.cpp:205-251
//   make_trace ......... S/trace.cpp:50-76
//   temperature_counts . S/dataset.cpp:39-52, build_epoch_index :61-83
//   synth_generate ..... S/dataset.cpp:121-247 (Morse clusters, default table)
//   init_params ........ S/model.cpp:177-193
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "common.hpp"
#include "rng.hpp"

namespace lamm_b200 {
namespace {

thread_local std::string t_last_error;

struct Slot {
    std::int64_t sample, atoms, split, chunk_rank;
};

// Worker for each of the G*B entries of one mini-batch: entries visited by
// descending key (ties by position: a stable sort), each given to the
// least-loaded worker that still has room; load ties go to the lower worker.
// Key = the atom count (the reference's balancer) or a predicted cost (double).
template <class Key>
void balance_minibatch(const Key* key, std::int64_t count, int G, int B, std::int32_t* worker) {
    // scratch reused across the epoch's mini-batches (plan() calls this ~n / (G B) times)
    thread_local std::vector<std::pair<Key, std::int64_t>> order;
    thread_local std::vector<Key> load;
    thread_local std::vector<int> filled;
    order.resize(static_cast<std::size_t>(count));
    for (std::int64_t e = 0; e < count; ++e) order[static_cast<std::size_t>(e)] = {key[e], e};
    std::sort(order.begin(), order.end(), [](const std::pair<Key, std::int64_t>& a, const std::pair<Key, std::int64_t>& b) {
        return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
    load.assign(static_cast<std::size_t>(G), Key(0));
    filled.assign(static_cast<std::size_t>(G), 0);
    for (const auto& oe : order) {
        const std::int64_t e = oe.second;
        int pick = -1;
        for (int g = 0; g < G; ++g)
            if (filled[g] < B && (pick < 0 || load[g] < load[pick])) pick = g;
        worker[e] = pick;
        load[pick] += key[e];
        ++filled[pick];
    }
}

struct PlanOut {
    std::int64_t* sample;
    std::int32_t* worker;
    std::int64_t* atoms;
    std::int64_t* split;
    std::int64_t* chunk_rank;
    std::int64_t* worker_atoms;
    double* worker_cost = nullptr;  // cost plans: predicted per-worker cost [batch][G] (nullable)
    const double* cost = nullptr;
    std::int64_t written = 0;
    std::int64_t batches = 0;
};

// pack_batch semantics (S/scheduler.cpp:43-58): worker-major, entry order
// preserved inside each worker.
void emit_minibatch(const std::vector<Slot>& mb, const std::vector<std::int32_t>& assign, int G, PlanOut& out) {
    std::int64_t* wa = out.worker_atoms + out.batches * G;
    double* wc = out.worker_cost ? out.worker_cost + out.batches * G : nullptr;
    for (int g = 0; g < G; ++g) {
        wa[g] = 0;
        if (wc) wc[g] = 0.0;
        for (std::size_t e = 0; e < mb.size(); ++e) {
            if (assign[e] != g) continue;
            const std::int64_t w = out.written++;
            out.sample[w] = mb[e].sample;
            out.worker[w] = g;
            out.atoms[w] = mb[e].atoms;
            out.split[w] = mb[e].split;
            out.chunk_rank[w] = mb[e].chunk_rank;
            wa[g] += mb[e].atoms;
            if (wc) wc[g] += out.cost[mb[e].sample];
        }
    }
    ++out.batches;
}

std::vector<std::int64_t> shuffled_ids(std::int64_t n, std::uint64_t seed) {
    std::vector<std::int64_t> ids(static_cast<std::size_t>(n));
    std::iota(ids.begin(), ids.end(), 0);
    Stream(seed).fisher_yates(ids);
    return ids;
}

}  // namespace

void set_last_error(const std::string& msg) { t_last_error = msg; }
const char* last_error_cstr() { return t_last_error.c_str(); }

}  // namespace lamm_b200

using namespace lamm_b200;

LAMM_API const char* lamm_last_error(void) { return last_error_cstr(); }

LAMM_API uint64_t lamm_mix_seed(uint64_t a, uint64_t b) { return splitmix_mix(a, b); }

LAMM_API int lamm_rng_normals(uint64_t seed, int64_t n, double* out) {
    return lamm_guard([&] {
        Stream s(seed);
        for (int64_t k = 0; k < n; ++k) out[k] = s.gauss();
    });
}

LAMM_API int lamm_greedy_assign(const int64_t* atoms, int64_t n, int32_t workers, int32_t batch_per_worker,
                                int32_t* worker_out) {
    return lamm_guard([&] {
        require(workers >= 1 && batch_per_worker >= 1, "greedy_assign: bad worker shape");
        require(n == static_cast<int64_t>(workers) * batch_per_worker,
                "greedy_assign: need exactly workers*batch_per_worker samples");
        balance_minibatch(atoms, n, workers, batch_per_worker, worker_out);
    });
}

namespace lamm_b200 {
namespace {
// plan() of S/scheduler.cpp:91-203 with the balancing key `key` (atoms: the
// reference's plan, bit-exact; a predicted per-sample cost: the cost plan).
template <class Key>
void plan_impl(const Key* key, const int64_t* atoms, int64_t n, int32_t G, int32_t B, int32_t S, uint64_t seed,
               int32_t mode, PlanOut& out, int64_t* n_batches, int64_t* dropped) {
    require(G >= 1, "schedule: workers must be >= 1");
    require(B >= 1, "schedule: batch_per_worker must be >= 1");
    require(S >= 1, "schedule: num_splits must be >= 1");
    require(mode >= 0 && mode <= 2, "schedule: unknown mode");
    for (int64_t k = 0; k < n; ++k) require(atoms[k] >= 1, "schedule: atom counts must be >= 1");
    const int64_t per_batch = static_cast<int64_t>(G) * B;
    const auto ids = shuffled_ids(n, seed);
    std::vector<Slot> mb;
    std::vector<Key> mb_key(static_cast<std::size_t>(per_batch));
    std::vector<std::int32_t> assign(static_cast<std::size_t>(per_batch));
    int64_t lost = 0;
    auto flush = [&] {
        for (std::size_t e = 0; e < mb.size(); ++e) mb_key[e] = key[mb[e].sample];
        if (mode == 2) {
            for (int64_t e = 0; e < per_batch; ++e) assign[static_cast<std::size_t>(e)] = static_cast<int32_t>(e / B);
        } else {
            balance_minibatch(mb_key.data(), per_batch, G, B, assign.data());
        }
        emit_minibatch(mb, assign, G, out);
        mb.clear();
    };
    if (mode == 0) {
        // (1) near-equal contiguous splits of the shuffled ids, each sorted
        //     by key descending (ties: lower id first).
        std::vector<int64_t> bounds(static_cast<std::size_t>(S) + 1, 0);
        for (int64_t s = 0; s < S; ++s) bounds[s + 1] = bounds[s] + n / S + (s < n % S ? 1 : 0);
        std::vector<std::int64_t> sorted = ids;
        int64_t ranks_max = 0;
        std::vector<std::pair<Key, std::int64_t>> kv;  // (key, id) pairs: the sort touches contiguous memory
        for (int64_t s = 0; s < S; ++s) {
            kv.resize(static_cast<std::size_t>(bounds[s + 1] - bounds[s]));
            for (int64_t k = bounds[s]; k < bounds[s + 1]; ++k) {
                const std::int64_t id = sorted[static_cast<std::size_t>(k)];
                kv[static_cast<std::size_t>(k - bounds[s])] = {key[id], id};
            }
            std::sort(kv.begin(), kv.end(), [](const std::pair<Key, std::int64_t>& a, const std::pair<Key, std::int64_t>& b) {
                return a.first != b.first ? a.first > b.first : a.second < b.second;
            });
            for (int64_t k = bounds[s]; k < bounds[s + 1]; ++k)
                sorted[static_cast<std::size_t>(k)] = kv[static_cast<std::size_t>(k - bounds[s])].second;
            const int64_t len = bounds[s + 1] - bounds[s];
            lost += len % G;
            ranks_max = std::max<int64_t>(ranks_max, len / G);
        }
        // (2) G-sized chunks consumed in transpose order (rank-major over
        // splits); (3) every B consecutive chunks form one mini-batch.
        for (int64_t r = 0; r < ranks_max; ++r)
            for (int64_t s = 0; s < S; ++s) {
                if ((r + 1) * G > bounds[s + 1] - bounds[s]) continue;
                for (int64_t k = r * G; k < (r + 1) * G; ++k) {
                    const std::int64_t id = sorted[static_cast<std::size_t>(bounds[s] + k)];
                    mb.push_back({id, atoms[id], s, r});
                }
                if (static_cast<int64_t>(mb.size()) == per_batch) flush();
            }
        lost += static_cast<int64_t>(mb.size());
        mb.clear();
    } else {
        const int64_t full = n / per_batch;
        lost = n - full * per_batch;
        for (int64_t b = 0; b < full; ++b) {
            for (int64_t e = 0; e < per_batch; ++e) {
                const std::int64_t id = ids[static_cast<std::size_t>(b * per_batch + e)];
                mb.push_back({id, atoms[id], 0, (b * per_batch + e) / G});
            }
            flush();
        }
    }
    *n_batches = out.batches;
    *dropped = lost;
}
}  // namespace
}  // namespace lamm_b200

LAMM_API int lamm_plan(const int64_t* atoms, int64_t n, int32_t G, int32_t B, int32_t S, uint64_t seed, int32_t mode,
                       int64_t* sample, int32_t* worker, int64_t* atoms_out, int64_t* split, int64_t* chunk_rank,
                       int64_t* worker_atoms, int64_t* n_batches, int64_t* dropped) {
    return lamm_guard([&] {
        PlanOut out{sample, worker, atoms_out, split, chunk_rank, worker_atoms};
        plan_impl(atoms, atoms, n, G, B, S, seed, mode, out, n_batches, dropped);
    });
}

LAMM_API int lamm_sample_cost(const int64_t* atoms, const int64_t* edges, int64_t n, const lamm_cost_model* cm,
                              double* cost) {
    return lamm_guard([&] {
        require(atoms && cm && cost, "sample_cost: null argument");
        require(std::isfinite(cm->per_sample) && std::isfinite(cm->per_atom) && std::isfinite(cm->per_edge),
                "cost model: non-finite coefficient");
        require(cm->per_edge == 0.0 || edges != nullptr, "cost model: per_edge set but no edge counts");
        for (int64_t k = 0; k < n; ++k) {
            // fixed order: ((per_sample + per_atom * atoms) + per_edge * edges)
            double c = cm->per_sample + cm->per_atom * static_cast<double>(atoms[k]);
            if (edges) c += cm->per_edge * static_cast<double>(edges[k]);
            require(c > 0.0, "cost model: predicted sample cost must be positive");
            cost[k] = c;
        }
    });
}

LAMM_API int lamm_plan_cost(const int64_t* atoms, const int64_t* edges, int64_t n, const lamm_cost_model* cm,
                            int32_t G, int32_t B, int32_t S, uint64_t seed, int32_t mode, int64_t* sample,
                            int32_t* worker, int64_t* atoms_out, int64_t* split, int64_t* chunk_rank,
                            int64_t* worker_atoms, double* worker_cost, int64_t* n_batches, int64_t* dropped) {
    return lamm_guard([&] {
        std::vector<double> cost(static_cast<std::size_t>(std::max<int64_t>(n, 1)));
        const int st = lamm_sample_cost(atoms, edges, n, cm, cost.data());
        if (st != 0) throw InputErr(last_error_cstr());
        PlanOut out{sample, worker, atoms_out, split, chunk_rank, worker_atoms};
        out.worker_cost = worker_cost;
        out.cost = cost.data();
        plan_impl(cost.data(), atoms, n, G, B, S, seed, mode, out, n_batches, dropped);
    });
}

LAMM_API int lamm_schedule_metrics(int64_t nb, int32_t G, int32_t B, const int32_t* worker, const int64_t* atoms,
                                   const int64_t* split, const int64_t* chunk_rank, double* max_imbalance,
                                   double* mean_imbalance, int64_t* monotonicity_violations,
                                   int64_t* growth_events) {
    return lamm_guard([&] {
        require(G >= 1 && B >= 1, "schedule_metrics: bad shape");
        const int64_t per = static_cast<int64_t>(G) * B;
        std::vector<int64_t> peak(static_cast<std::size_t>(G), 0), totals(static_cast<std::size_t>(G));
        double worst = 0.0, acc = 0.0;
        int64_t growth = 0;
        for (int64_t st = 0; st < nb; ++st) {
            std::fill(totals.begin(), totals.end(), 0);
            for (int64_t e = 0; e < per; ++e) totals[worker[st * per + e]] += atoms[st * per + e];
            int64_t sum = 0, top = 0;
            for (int g = 0; g < G; ++g) {
                sum += totals[g];
                top = std::max(top, totals[g]);
                if (totals[g] > peak[g]) {
                    ++growth;
                    peak[g] = totals[g];
                }
            }
            const double mean = static_cast<double>(sum) / static_cast<double>(G);
            const double ratio = mean > 0.0 ? static_cast<double>(top) / mean : 1.0;
            worst = std::max(worst, ratio);
            acc += ratio;
        }
        if (nb > 0) {
            acc /= static_cast<double>(nb);
        } else {
            worst = acc = 1.0;
        }
        // Chunk totals keyed by (split, chunk_rank), walked in key order: the entries
        // ordered by (split, rank) with a two-pass LSD counting sort (stable by rank,
        // then by split), O(n) instead of a comparison sort of the whole epoch.
        const int64_t m = nb * per;
        int64_t max_split = 0, max_rank = 0;
        for (int64_t e = 0; e < m; ++e) {
            require(split[e] >= 0 && chunk_rank[e] >= 0, "schedule_metrics: negative split / chunk rank");
            max_split = std::max(max_split, split[e]);
            max_rank = std::max(max_rank, chunk_rank[e]);
        }
        auto counting = [&](const std::vector<int64_t>& in, const int64_t* key, int64_t kmax) {
            std::vector<int64_t> start(static_cast<std::size_t>(kmax) + 2, 0), out(in.size());
            for (const int64_t e : in) ++start[static_cast<std::size_t>(key[e]) + 1];
            for (int64_t k = 0; k <= kmax; ++k) start[k + 1] += start[k];
            for (const int64_t e : in) out[static_cast<std::size_t>(start[static_cast<std::size_t>(key[e])]++)] = e;
            return out;
        };
        std::vector<int64_t> order(static_cast<std::size_t>(m));
        std::iota(order.begin(), order.end(), 0);
        order = counting(counting(order, chunk_rank, max_rank), split, max_split);
        int64_t violations = 0, prev_split = -1, prev_total = 0;
        for (std::size_t e = 0; e < order.size();) {
            const int64_t s0 = split[order[e]], r0 = chunk_rank[order[e]];
            std::size_t f = e;
            int64_t total = 0;
            while (f < order.size() && split[order[f]] == s0 && chunk_rank[order[f]] == r0) total += atoms[order[f++]];
            if (s0 == prev_split && total > prev_total) ++violations;
            prev_split = s0;
            prev_total = total;
            e = f;
        }
        *max_imbalance = worst;
        *mean_imbalance = acc;
        *monotonicity_violations = violations;
        *growth_events = growth;
    });
}

namespace lamm_b200 {
namespace {
int64_t lognormal_count(double mode, double sigma, Stream& s) {
    const double mu = std::log(mode) + sigma * sigma;  // mode = exp(mu - sigma^2)
    return std::llround(std::exp(s.gauss(mu, sigma)));
}
}  // namespace
}  // namespace lamm_b200

LAMM_API int lamm_make_trace(int32_t kind, int64_t count, int64_t lo, int64_t hi, double constant_atoms, double mode,
                             double sigma, double mode_a, double sigma_a, double mode_b, double sigma_b,
                             double weight_a, uint64_t seed, int64_t* out) {
    return lamm_guard([&] {
        require(count >= 1, "trace: count must be >= 1");
        require(lo >= 1 && hi >= lo, "trace: bad atom bounds");
        require(constant_atoms >= 1.0 && mode >= 1.0 && mode_a >= 1.0 && mode_b >= 1.0, "trace: modes must be >= 1");
        require(sigma > 0.0 && sigma_a > 0.0 && sigma_b > 0.0, "trace: sigmas must be positive");
        require(weight_a >= 0.0 && weight_a <= 1.0, "trace: weight_a must be in [0, 1]");
        require(kind >= 0 && kind <= 3, "trace: unknown kind");
        Stream s(seed);
        for (int64_t k = 0; k < count; ++k) {
            int64_t v;
            if (kind == 0) v = std::llround(constant_atoms);
            else if (kind == 1) v = lo + static_cast<int64_t>(s.below(static_cast<uint64_t>(hi - lo + 1)));
            else if (kind == 2) v = lognormal_count(mode, sigma, s);
            else v = s.unit() < weight_a ? lognormal_count(mode_a, sigma_a, s) : lognormal_count(mode_b, sigma_b, s);
            out[k] = std::clamp(v, lo, hi);
        }
    });
}

LAMM_API int lamm_temperature_counts(const double* sizes, int32_t k, double T, double* out) {
    return lamm_guard([&] {
        require(k >= 1, "temperature_counts: no subset sizes");
        require(T >= 1.0, "temperature_counts: temperature must be >= 1");
        double largest = 0.0;
        for (int32_t q = 0; q < k; ++q) {
            require(sizes[q] > 0.0, "temperature_counts: sizes must be positive");
            largest = std::max(largest, sizes[q]);
        }
        const double inv_t = 1.0 / T;
        for (int32_t q = 0; q < k; ++q) out[q] = std::pow(largest, 1.0 - inv_t) * std::pow(sizes[q], inv_t);
    });
}

LAMM_API int lamm_build_epoch_index(const double* repeats, const int64_t* sizes, int32_t k, uint64_t seed,
                                    int64_t cap, int32_t* out_subset, int64_t* out_sample, int64_t* count) {
    return lamm_guard([&] {
        std::vector<std::pair<int32_t, int64_t>> entries;
        for (int32_t q = 0; q < k; ++q) {
            require(sizes[q] > 0, "build_epoch_index: subset sizes must be positive");
            const int64_t total = std::llround(repeats[q]);
            require(total >= 0, "build_epoch_index: negative repeat count");
            const int64_t base = total / sizes[q], extra = total % sizes[q];
            for (int64_t s = 0; s < sizes[q]; ++s)
                for (int64_t c = 0; c < base + (s < extra ? 1 : 0); ++c) entries.emplace_back(q, s);
        }
        Stream(seed).fisher_yates(entries);
        *count = static_cast<int64_t>(entries.size());
        for (int64_t e = 0; e < std::min<int64_t>(cap, *count); ++e) {
            out_subset[e] = entries[static_cast<std::size_t>(e)].first;
            out_sample[e] = entries[static_cast<std::size_t>(e)].second;
        }
    });
}

// ---------------------------------------------------------------- synth --
namespace lamm_b200 {
namespace {
constexpr double kMorseDepth = 1.0, kMorseStiffness = 2.2, kMorseReq = 1.9;  // H/dataset.hpp:90-94

inline double len3(double x, double y, double z) { return std::sqrt(x * x + y * y + z * z); }

int atom_count(double mode, double sigma, int lo, int hi, Stream& s) {
    const double mu = std::log(mode) + sigma * sigma;
    return std::clamp(static_cast<int>(std::llround(std::exp(s.gauss(mu, sigma)))), lo, hi);
}

// Pair forces of the all-pairs Morse surface; f is [n][3].
void morse_grad(int n, const double* x, double* f) {
    std::fill(f, f + 3 * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            const double dx = x[3 * i] - x[3 * j], dy = x[3 * i + 1] - x[3 * j + 1], dz = x[3 * i + 2] - x[3 * j + 2];
            const double r = len3(dx, dy, dz);
            const double e = std::exp(-kMorseStiffness * (r - kMorseReq));
            const double dvdr = 2.0 * kMorseDepth * (1.0 - e) * kMorseStiffness * e;
            const double s = -dvdr / r;
            const double fx = s * dx, fy = s * dy, fz = s * dz;
            f[3 * i] = f[3 * i] + fx, f[3 * i + 1] = f[3 * i + 1] + fy, f[3 * i + 2] = f[3 * i + 2] + fz;
            f[3 * j] = f[3 * j] - fx, f[3 * j + 1] = f[3 * j + 1] - fy, f[3 * j + 2] = f[3 * j + 2] - fz;
        }
}

double morse_total(int n, const double* x) {
    double e = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            const double r = len3(x[3 * i] - x[3 * j], x[3 * i + 1] - x[3 * j + 1], x[3 * i + 2] - x[3 * j + 2]);
            const double g = 1.0 - std::exp(-kMorseStiffness * (r - kMorseReq));
            e += kMorseDepth * (g * g - 1.0);
        }
    return e;
}

struct SynthArgs {
    int task;
    double mode, sigma;
    int lo, hi;
    const int32_t* elements;
    int n_elements;
    int relax_steps;
    double relax_step, energy_scale;
    const int32_t* off_z;
    const double* off_v;
    int n_off;
    uint64_t seed;
};

void synth_one(const SynthArgs& a, int64_t s, double* x, int32_t* z, uint8_t* em, uint8_t* fm, double* energy,
               double* f) {
    Stream st(splitmix_mix(a.seed, static_cast<uint64_t>(s)));
    const int n = atom_count(a.mode, a.sigma, a.lo, a.hi, st);
    // random_cluster: rejection-sample points in a ball with a minimum
    // separation, growing the ball by 10% after 200 failed placements.
    const double min_sep = 0.8 * kMorseReq;
    double radius = 0.75 * kMorseReq * std::cbrt(static_cast<double>(n));
    for (int at = 0; at < n; ++at) {
        double px, py, pz;
        for (int attempt = 0;; ++attempt) {
            px = st.in(-radius, radius);
            py = st.in(-radius, radius);
            pz = st.in(-radius, radius);
            if (len3(px, py, pz) > radius) continue;
            bool clear = true;
            for (int q = 0; q < at && clear; ++q)
                clear = !(len3(px - x[3 * q], py - x[3 * q + 1], pz - x[3 * q + 2]) < min_sep);
            if (clear) break;
            if (attempt >= 200) {
                radius *= 1.1;
                attempt = 0;
            }
        }
        x[3 * at] = px, x[3 * at + 1] = py, x[3 * at + 2] = pz;
        z[at] = a.elements[st.below(static_cast<uint64_t>(a.n_elements))];
    }
    // relax: damped steepest descent with a 0.25 A per-atom move cap.
    for (int step = 0; step < a.relax_steps; ++step) {
        morse_grad(n, x, f);
        for (int at = 0; at < n; ++at) {
            double mx = a.relax_step * f[3 * at], my = a.relax_step * f[3 * at + 1], mz = a.relax_step * f[3 * at + 2];
            const double m = len3(mx, my, mz);
            if (m > 0.25) {
                const double sc = 0.25 / m;
                mx = sc * mx, my = sc * my, mz = sc * mz;
            }
            x[3 * at] = x[3 * at] + mx, x[3 * at + 1] = x[3 * at + 1] + my, x[3 * at + 2] = x[3 * at + 2] + mz;
        }
    }
    *em = 0, *fm = 0, *energy = 0.0;
    std::fill(f, f + 3 * n, 0.0);
    if (a.task == 2) return;
    double e = a.energy_scale * morse_total(n, x);
    for (int at = 0; at < n; ++at)
        for (int q = 0; q < a.n_off; ++q)
            if (a.off_z[q] == z[at]) {
                e += a.off_v[q];
                break;
            }
    *energy = e;
    *em = 1;
    if (a.task == 0) {
        morse_grad(n, x, f);
        for (int k = 0; k < 3 * n; ++k) f[k] = a.energy_scale * f[k];
        *fm = 1;
    }
}
}  // namespace
}  // namespace lamm_b200

LAMM_API int lamm_synth_counts(int64_t count, double mode, double sigma, int32_t lo, int32_t hi, uint64_t seed,
                               int64_t* atom_ptr) {
    return lamm_guard([&] {
        require(count >= 0, "synth_generate: negative count");
        require(lo >= 1 && hi >= lo, "synth_generate: bad atom-count bounds");
        require(mode >= 1.0, "synth_generate: atom_count_mode must be >= 1");
        atom_ptr[0] = 0;
        for (int64_t s = 0; s < count; ++s) {
            Stream st(splitmix_mix(seed, static_cast<uint64_t>(s)));
            atom_ptr[s + 1] = atom_ptr[s] + atom_count(mode, sigma, lo, hi, st);
        }
    });
}

LAMM_API int lamm_synth_fill(int32_t task, int64_t count, double mode, double sigma, int32_t lo, int32_t hi,
                             const int32_t* elements, int32_t n_elements, int32_t relax_steps, double relax_step,
                             double energy_scale, const int32_t* off_z, const double* off_v, int32_t n_off,
                             uint64_t seed, int32_t threads, const int64_t* atom_ptr, double* positions,
                             int32_t* atomic_numbers, uint8_t* energy_mask, uint8_t* force_mask, double* energy,
                             double* forces) {
    return lamm_guard([&] {
        require(n_elements >= 1, "synth_generate: element list is empty");
        for (int32_t q = 0; q < n_elements; ++q)
            require(elements[q] >= 1 && elements[q] <= 118, "synth_generate: atomic number out of range");
        require(task >= 0 && task <= 2, "synth_generate: unknown task");
        const SynthArgs a{task,     mode,       sigma,        lo,    hi,    elements, n_elements, relax_steps,
                          relax_step, energy_scale, off_z, off_v, n_off, seed};
        auto run = [&](int64_t s) {
            synth_one(a, s, positions + 3 * atom_ptr[s], atomic_numbers + atom_ptr[s], energy_mask + s,
                      force_mask + s, energy + s, forces + 3 * atom_ptr[s]);
        };
        const int nt = std::max(1, std::min<int>(threads, static_cast<int>(std::max<int64_t>(count, 1))));
        if (nt == 1) {
            for (int64_t s = 0; s < count; ++s) run(s);
        } else {
            std::vector<std::thread> pool;
            for (int t = 0; t < nt; ++t)
                pool.emplace_back([&, t] {
                    for (int64_t s = t; s < count; s += nt) run(s);
                });
            for (auto& th : pool) th.join();
        }
    });
}

LAMM_API int64_t lamm_param_count(const lamm_model_config* c) {
    if (!c) return -1;
    const int64_t H = c->hidden, L = c->layers, K = c->rbf, D = c->heads;
    return 118 * H + L * H * K + L * H * H + H * D + (2 * H + K) * D;
}

LAMM_API int lamm_init_params(const lamm_model_config* c, uint64_t seed, double* out) {
    return lamm_guard([&] {
        require(c != nullptr, "init_params: null config");
        require(c->hidden >= 1, "model: hidden must be >= 1");
        require(c->layers >= 0, "model: layers must be >= 0");
        require(c->rbf >= 2, "model: rbf must be >= 2");
        require(c->cutoff > 0.0, "model: cutoff must be positive");
        require(c->heads >= 1, "model: heads must be >= 1");
        const int64_t H = c->hidden, L = c->layers, K = c->rbf, D = c->heads;
        Stream st(seed);
        int64_t o = 0;
        auto fill = [&](int64_t count, double scale) {
            for (int64_t k = 0; k < count; ++k) out[o++] = st.in(-scale, scale);
        };
        fill(118 * H, 1.0);
        for (int64_t l = 0; l < L; ++l) fill(H * K, 1.0 / std::sqrt(static_cast<double>(K)));
        for (int64_t l = 0; l < L; ++l) fill(H * H, 1.0 / std::sqrt(static_cast<double>(H)));
        fill(H * D, 1.0 / std::sqrt(static_cast<double>(H)));
        fill((2 * H + K) * D, 1.0 / std::sqrt(static_cast<double>(2 * H + K)));
    });
}

// simulator::simulate (S/simulator.cpp:19-59): per step and worker compute =
// alpha + beta * atoms, + delta when the worker's atoms exceed its running high
// water; step = slowest worker + gamma. Bit-exact with the reference (the same
// operations in the same order). worker_cost (nullable): a predicted per-worker
// cost [n_batches][G] in seconds (lamm_plan_cost's worker_cost scaled) used in
// place of alpha + beta * atoms (extension: the cost model's own prediction).
LAMM_API int lamm_simulate(const int64_t* worker_atoms, const double* worker_cost, int64_t n_batches, int32_t G,
                           int64_t samples_per_batch, const lamm_sim_cost* cost, double* step_time,
                           double* step_idle, int32_t* step_realloc, int64_t* step_max_atoms, double* worker_idle,
                           lamm_sim_totals* totals) {
    return lamm_guard([&] {
        require(worker_atoms && cost && totals, "simulate: null argument");
        const double v[] = {cost->alpha_s, cost->beta_s_per_atom, cost->gamma_s, cost->delta_s};
        for (double x : v)
            require(x >= 0.0 && std::isfinite(x), "cost model: coefficients must be finite and non-negative");
        require(cost->alpha_s + cost->beta_s_per_atom > 0.0, "cost model: compute cost must be positive");
        require(G >= 1, "simulate: schedule has no workers");
        std::vector<int64_t> peak(static_cast<std::size_t>(G), 0);
        std::vector<double> busy(static_cast<std::size_t>(G)), idle_acc(static_cast<std::size_t>(G), 0.0);
        double total = 0.0;
        int64_t reallocs = 0, samples = 0;
        for (int64_t b = 0; b < n_batches; ++b) {
            double slowest = 0.0, idle = 0.0;
            int32_t rec_realloc = 0;
            int64_t max_atoms = 0;
            for (int g = 0; g < G; ++g) {
                const int64_t atoms = worker_atoms[b * G + g];
                double t = worker_cost ? worker_cost[b * G + g]
                                       : cost->alpha_s + cost->beta_s_per_atom * static_cast<double>(atoms);
                if (atoms > peak[g]) {
                    t += cost->delta_s;
                    peak[g] = atoms;
                    ++rec_realloc;
                }
                busy[g] = t;
                slowest = std::max(slowest, t);
                max_atoms = std::max(max_atoms, atoms);
            }
            const double st = slowest + cost->gamma_s;
            for (int g = 0; g < G; ++g) {
                const double i = slowest - busy[g];
                idle_acc[g] += i;
                idle += i;
            }
            reallocs += rec_realloc;
            total += st;
            samples += samples_per_batch;
            if (step_time) step_time[b] = st;
            if (step_idle) step_idle[b] = idle;
            if (step_realloc) step_realloc[b] = rec_realloc;
            if (step_max_atoms) step_max_atoms[b] = max_atoms;
        }
        if (worker_idle) std::copy(idle_acc.begin(), idle_acc.end(), worker_idle);
        totals->total_s = total;
        totals->realloc_events = reallocs;
        totals->samples = samples;
        totals->throughput_samples_per_s = total > 0.0 ? static_cast<double>(samples) / total : 0.0;
    });
}
