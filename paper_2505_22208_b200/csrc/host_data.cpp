// host_data.cpp - the data layer around the train step, host side: the pieces of
// the reference's orchestration (S/trainer.cpp:64-125, S/loss.cpp:17-111,
// S/dataset.cpp:85-111, S/denoise.cpp:7-40, S/model.cpp:167-202) that the
// B200 trainer (include/lamm_b200_trainer.hpp) needs once per run or per report,
// re-implemented so the product links no reference code:
//   filter_max_atoms / split_train_val ... S/dataset.cpp:85-111 (bit-exact)
//   apply_noise ........................... S/denoise.cpp:7-40   (bit-exact draws)
//   estimate_pseudo_force_std ............. S/trainer.cpp:82-100 (bit-exact)
//   fit_reference / fit_normalizer ........ S/loss.cpp:17-111    (minimum-norm least
//        squares by a complete orthogonal decomposition written here: Householder QR
//        with column pivoting, rank by |R_kk| > eps * min(m, n) * |R_00| (Eigen's
//        COD default), then a QR of the rank rows' transpose; within 1e-9 relative of
//        an SVD minimum-norm solve, tests/test_data_layer.py)
//   init_heads / reset_heads .............. S/model.cpp:167-202  (bit-exact)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "common.hpp"
#include "rng.hpp"

namespace lamm_b200 {
namespace {

constexpr std::uint64_t kProbeTag = 0x50535444;  // S/trainer.cpp:26

// S/denoise.cpp:7-40: raw draws Rng(seed).normal(0, sigma) per atom x, y, z;
// centered: minus their mean (sequential Vec3 sum, then (1/n) * sum); noisy =
// x + effective, pseudo force = -1 * effective.
void noise_one(const double* pos, int64_t n, double sigma, int scheme, std::uint64_t seed, double* noisy,
               double* pseudo) {
    Stream st(seed);
    std::vector<double> eff(static_cast<std::size_t>(3 * n));
    for (int64_t k = 0; k < 3 * n; ++k) eff[k] = st.gauss(0.0, sigma);
    if (scheme == 1) {
        double m[3] = {0.0, 0.0, 0.0};
        for (int64_t a = 0; a < n; ++a)
            for (int c = 0; c < 3; ++c) m[c] = m[c] + eff[3 * a + c];
        const double inv = 1.0 / static_cast<double>(n);
        for (int c = 0; c < 3; ++c) m[c] = inv * m[c];
        for (int64_t a = 0; a < n; ++a)
            for (int c = 0; c < 3; ++c) eff[3 * a + c] = eff[3 * a + c] - m[c];
    }
    for (int64_t k = 0; k < 3 * n; ++k) {
        if (noisy) noisy[k] = pos[k] + eff[k];
        if (pseudo) pseudo[k] = -1.0 * eff[k];
    }
}

// Minimum-norm least squares min ||A x - b||, A m x n (row-major), by a complete
// orthogonal decomposition: A P = Q [R11 R12; 0 0] (Householder, column pivoting),
// then [R11 R12]^T = Z [T; 0]; x = P Z [T^-T (Q^T b)_r; 0].
std::vector<double> min_norm_lstsq(std::vector<double> A, std::vector<double> b, int64_t m, int64_t n) {
    const int64_t kmax = std::min(m, n);
    std::vector<int64_t> perm(static_cast<std::size_t>(n));
    for (int64_t j = 0; j < n; ++j) perm[j] = j;
    auto at = [&](int64_t i, int64_t j) -> double& { return A[static_cast<std::size_t>(i * n + j)]; };
    std::vector<double> rdiag(static_cast<std::size_t>(kmax), 0.0);
    for (int64_t k = 0; k < kmax; ++k) {
        // pivot: the remaining column of largest norm (ties: the lower index)
        int64_t best = k;
        double bn = -1.0;
        for (int64_t j = k; j < n; ++j) {
            double s = 0.0;
            for (int64_t i = k; i < m; ++i) s += at(i, j) * at(i, j);
            if (s > bn) bn = s, best = j;
        }
        if (best != k) {
            for (int64_t i = 0; i < m; ++i) std::swap(at(i, k), at(i, best));
            std::swap(perm[k], perm[best]);
        }
        const double norm = std::sqrt(bn);
        if (norm == 0.0) {
            rdiag[k] = 0.0;
            continue;
        }
        const double alpha = at(k, k) >= 0.0 ? -norm : norm;
        // v = x - alpha e1, H = I - 2 v v^T / (v^T v)
        std::vector<double> v(static_cast<std::size_t>(m - k));
        for (int64_t i = k; i < m; ++i) v[i - k] = at(i, k);
        v[0] -= alpha;
        double vv = 0.0;
        for (double x : v) vv += x * x;
        if (vv > 0.0) {
            for (int64_t j = k; j < n; ++j) {
                double s = 0.0;
                for (int64_t i = k; i < m; ++i) s += v[i - k] * at(i, j);
                s = 2.0 * s / vv;
                for (int64_t i = k; i < m; ++i) at(i, j) -= s * v[i - k];
            }
            double s = 0.0;
            for (int64_t i = k; i < m; ++i) s += v[i - k] * b[i];
            s = 2.0 * s / vv;
            for (int64_t i = k; i < m; ++i) b[i] -= s * v[i - k];
        }
        rdiag[k] = at(k, k);
    }
    // numerical rank (Eigen's COD default threshold)
    const double thr = std::numeric_limits<double>::epsilon() * static_cast<double>(kmax);
    int64_t r = 0;
    const double r00 = kmax > 0 ? std::fabs(rdiag[0]) : 0.0;
    while (r < kmax && std::fabs(rdiag[r]) > thr * r00) ++r;
    std::vector<double> y(static_cast<std::size_t>(n), 0.0);
    if (r > 0) {
        // M = [R11 R12]^T (n x r), QR of M without pivoting: M = Z [T; 0]
        std::vector<double> M(static_cast<std::size_t>(n * r));
        auto mt = [&](int64_t i, int64_t j) -> double& { return M[static_cast<std::size_t>(i * r + j)]; };
        for (int64_t i = 0; i < r; ++i)
            for (int64_t j = 0; j < n; ++j) mt(j, i) = j >= i ? at(i, j) : 0.0;
        std::vector<std::vector<double>> vs(static_cast<std::size_t>(r));
        std::vector<double> vvs(static_cast<std::size_t>(r), 0.0);
        for (int64_t k = 0; k < r; ++k) {
            double s = 0.0;
            for (int64_t i = k; i < n; ++i) s += mt(i, k) * mt(i, k);
            const double norm = std::sqrt(s);
            const double alpha = mt(k, k) >= 0.0 ? -norm : norm;
            auto& v = vs[k];
            v.assign(static_cast<std::size_t>(n - k), 0.0);
            for (int64_t i = k; i < n; ++i) v[i - k] = mt(i, k);
            v[0] -= alpha;
            double vv = 0.0;
            for (double x : v) vv += x * x;
            vvs[k] = vv;
            if (vv > 0.0)
                for (int64_t j = k; j < r; ++j) {
                    double t = 0.0;
                    for (int64_t i = k; i < n; ++i) t += v[i - k] * mt(i, j);
                    t = 2.0 * t / vv;
                    for (int64_t i = k; i < n; ++i) mt(i, j) -= t * v[i - k];
                }
        }
        // T^T w = c (lower triangular), c = (Q^T b)[0:r]
        std::vector<double> w(static_cast<std::size_t>(n), 0.0);
        for (int64_t i = 0; i < r; ++i) {
            double s = b[i];
            for (int64_t j = 0; j < i; ++j) s -= mt(j, i) * w[j];
            w[i] = s / mt(i, i);
        }
        // y = Z [w; 0]: the reflectors applied in reverse
        for (int64_t k = r - 1; k >= 0; --k) {
            const auto& v = vs[k];
            if (vvs[k] <= 0.0) continue;
            double t = 0.0;
            for (int64_t i = k; i < n; ++i) t += v[i - k] * w[i];
            t = 2.0 * t / vvs[k];
            for (int64_t i = k; i < n; ++i) w[i] -= t * v[i - k];
        }
        y = w;
    }
    std::vector<double> x(static_cast<std::size_t>(n), 0.0);
    for (int64_t j = 0; j < n; ++j) x[perm[j]] = y[j];
    return x;
}

}  // namespace
}  // namespace lamm_b200

using namespace lamm_b200;

LAMM_API int lamm_filter_max_atoms(const int64_t* atom_ptr, int64_t n_samples, int64_t limit, int64_t* kept,
                                   int64_t* n_kept) {
    return lamm_guard([&] {
        require(atom_ptr && kept && n_kept, "filter_max_atoms: null argument");
        require(limit >= 1, "filter_max_atoms: limit must be >= 1");
        int64_t c = 0;
        for (int64_t s = 0; s < n_samples; ++s)
            if (atom_ptr[s + 1] - atom_ptr[s] <= limit) kept[c++] = s;
        *n_kept = c;
    });
}

LAMM_API int lamm_split_train_val(int64_t n, double val_fraction, uint64_t seed, int64_t* train, int64_t* n_train,
                                  int64_t* val, int64_t* n_val) {
    return lamm_guard([&] {
        require(n >= 0 && train && n_train && val && n_val, "split_train_val: bad argument");
        require(val_fraction >= 0.0 && val_fraction <= 1.0, "split_train_val: val_fraction must be in [0, 1]");
        std::vector<int64_t> perm(static_cast<std::size_t>(n));
        for (int64_t k = 0; k < n; ++k) perm[k] = k;
        Stream(seed).fisher_yates(perm);
        const int64_t nv = std::llround(val_fraction * static_cast<double>(n));
        std::vector<int64_t> v(perm.begin(), perm.begin() + nv), t(perm.begin() + nv, perm.end());
        std::sort(v.begin(), v.end());
        std::sort(t.begin(), t.end());
        std::copy(v.begin(), v.end(), val);
        std::copy(t.begin(), t.end(), train);
        *n_val = nv, *n_train = n - nv;
    });
}

LAMM_API int lamm_apply_noise(const double* positions, int64_t n_atoms, double sigma, int32_t scheme, uint64_t seed,
                              double* noisy, double* pseudo_forces) {
    return lamm_guard([&] {
        require(positions && n_atoms >= 1, "apply_displacements: system has no atoms");
        require(sigma > 0.0, "apply_noise: sigma must be positive");
        noise_one(positions, n_atoms, sigma, scheme, seed, noisy, pseudo_forces);
    });
}

LAMM_API int lamm_pseudo_force_std(const int64_t* atom_ptr, const double* positions, const int64_t* ids,
                                   int64_t n_ids, double sigma, int32_t scheme, uint64_t seed, double* out) {
    return lamm_guard([&] {
        require(atom_ptr && positions && out, "pseudo_force_std: null argument");
        require(sigma > 0.0, "apply_noise: sigma must be positive");
        const int64_t probe = std::min<int64_t>(n_ids, 256);
        double sum = 0.0, sq = 0.0;
        int64_t count = 0;
        std::vector<double> pf;
        for (int64_t v = 0; v < probe; ++v) {
            const int64_t s = ids ? ids[v] : v;
            const int64_t n = atom_ptr[s + 1] - atom_ptr[s];
            require(n >= 1, "apply_displacements: system has no atoms");
            pf.resize(static_cast<std::size_t>(3 * n));
            noise_one(positions + 3 * atom_ptr[s], n, sigma, scheme, splitmix_mix(seed, kProbeTag + v), nullptr,
                      pf.data());
            for (double c : pf) {
                sum += c;
                sq += c * c;
                ++count;
            }
        }
        if (count == 0) {
            *out = sigma;
            return;
        }
        const double mean = sum / static_cast<double>(count);
        *out = std::max(std::sqrt(std::max(sq / static_cast<double>(count) - mean * mean, 0.0)), 1e-8);
    });
}

LAMM_API int lamm_fit_normalizer(const lamm_batch_view* b, double pseudo_force_std, lamm_normalizer* out) {
    return lamm_guard([&] {
        require(b && out, "fit_normalizer: null argument");
        std::memset(out, 0, sizeof(lamm_normalizer));
        out->energy_mean = 0.0, out->energy_std = 1.0, out->force_std = 1.0;
        const int64_t B = b->n_samples;
        auto emask = [&](int64_t s) { return b->energy_mask && b->energy_mask[s]; };
        auto fmask = [&](int64_t s) { return b->force_mask && b->force_mask[s]; };
        int64_t n_energy = 0;
        for (int64_t s = 0; s < B; ++s) n_energy += emask(s) ? 1 : 0;
        if (n_energy > 0) {
            require(b->energy != nullptr, "fit_normalizer: energy mask set but energy missing");
            // S/loss.cpp:17-48: elements of the labelled samples in ascending Z, one
            // composition row per labelled sample
            bool present[119] = {};
            for (int64_t s = 0; s < B; ++s)
                if (emask(s))
                    for (int64_t a = b->atom_ptr[s]; a < b->atom_ptr[s + 1]; ++a) {
                        const int z = b->atomic_numbers[a];
                        require(z >= 1 && z <= 118, "atomic number outside [1, 118]");
                        present[z] = true;
                    }
            std::vector<int> order;
            for (int z = 1; z <= 118; ++z)
                if (present[z]) order.push_back(z);
            const int64_t m = n_energy, n = static_cast<int64_t>(order.size());
            std::vector<int> col(119, -1);
            for (int64_t c = 0; c < n; ++c) col[order[c]] = static_cast<int>(c);
            std::vector<double> A(static_cast<std::size_t>(m * n), 0.0), y(static_cast<std::size_t>(m));
            int64_t row = 0;
            for (int64_t s = 0; s < B; ++s) {
                if (!emask(s)) continue;
                for (int64_t a = b->atom_ptr[s]; a < b->atom_ptr[s + 1]; ++a) A[row * n + col[b->atomic_numbers[a]]] += 1.0;
                y[row++] = b->energy[s];
            }
            const auto rho = min_norm_lstsq(A, y, m, n);
            for (int64_t c = 0; c < n; ++c) out->rho[order[c]] = rho[c], out->rho_has[order[c]] = 1;
            // S/loss.cpp:64-89: residual mean and std, in sample order
            auto refsum = [&](int64_t s) {
                double t = 0.0;
                for (int64_t a = b->atom_ptr[s]; a < b->atom_ptr[s + 1]; ++a) t += out->rho[b->atomic_numbers[a]];
                return t;
            };
            double sum = 0.0;
            for (int64_t s = 0; s < B; ++s)
                if (emask(s)) sum += b->energy[s] - refsum(s);
            out->energy_mean = sum / static_cast<double>(n_energy);
            double sq = 0.0;
            for (int64_t s = 0; s < B; ++s) {
                if (!emask(s)) continue;
                const double r = b->energy[s] - refsum(s) - out->energy_mean;
                sq += r * r;
            }
            out->energy_std = std::max(std::sqrt(sq / static_cast<double>(n_energy)), 1e-8);
            out->has_energy_stats = 1;
        }
        // S/loss.cpp:91-110: per-component force std of the force-labelled samples
        int64_t n_comp = 0;
        double f_sum = 0.0;
        for (int64_t s = 0; s < B; ++s) {
            if (!fmask(s)) continue;
            require(b->forces != nullptr, "fit_normalizer: force mask set but forces missing");
            for (int64_t k = 3 * b->atom_ptr[s]; k < 3 * b->atom_ptr[s + 1]; ++k) f_sum += b->forces[k], ++n_comp;
        }
        if (n_comp > 0) {
            const double mean = f_sum / static_cast<double>(n_comp);
            double sq = 0.0;
            for (int64_t s = 0; s < B; ++s) {
                if (!fmask(s)) continue;
                for (int64_t k = 3 * b->atom_ptr[s]; k < 3 * b->atom_ptr[s + 1]; ++k)
                    sq += (b->forces[k] - mean) * (b->forces[k] - mean);
            }
            out->force_std = std::max(std::sqrt(sq / static_cast<double>(n_comp)), 1e-8);
        } else if (pseudo_force_std > 0.0) {
            out->force_std = pseudo_force_std;
        }
    });
}

LAMM_API int lamm_init_heads(const lamm_model_config* c, int32_t heads, uint64_t seed, double* energy_head,
                             double* force_head) {
    return lamm_guard([&] {
        require(c && energy_head && force_head, "init_heads: null argument");
        require(heads >= 1, "reset_heads: need at least one head");
        const int64_t H = c->hidden, K = c->rbf;
        Stream st(seed);
        const double se = 1.0 / std::sqrt(static_cast<double>(H)), sf = 1.0 / std::sqrt(static_cast<double>(2 * H + K));
        for (int64_t k = 0; k < H * heads; ++k) energy_head[k] = st.in(-se, se);
        for (int64_t k = 0; k < (2 * H + K) * heads; ++k) force_head[k] = st.in(-sf, sf);
    });
}
