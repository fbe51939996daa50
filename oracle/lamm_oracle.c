/*
 * oracle/lamm_oracle.c - plain-C restatement of LaMM's load-balanced
 * energy/force train step (the reference hot path), fp64 throughout.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity CHECKER: tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product (paper_2505_22208_b200/) never links, imports or calls it.
 *
 * Every function restates the reference algorithm with the same floating-point
 * operation order, so on x86-64 with glibc libm and no FMA contraction it is
 * BIT-IDENTICAL to the reference compiled in oracle/_ref. tests/test_oracle_pin.py
 * pins that claim on randomized inputs plus the SPEC known-answer cases and the
 * committed golden vectors in tests/golden/.
 *
 * Reference locations (H = /root/reference/proj/core/include/lamm,
 *                      S = /root/reference/proj/core/src):
 *   RNG ............ H/rng.hpp:18-81
 *   neighbour list . S/core.cpp:30-48
 *   model .......... S/model.cpp:17-110 (encoder), :177-193 (init), :208-253 (heads), :299-425 (backward)
 *   loss ........... S/loss.cpp:113-126 (normalize), :140-213 (Eq. 5)
 *   denoise ........ S/denoise.cpp:7-53
 *   train step ..... S/trainer.cpp:258-327, RMS optimizer :29-54
 *   scheduler ...... S/scheduler.cpp:43-251
 *   trace/dataset .. S/trace.cpp:50-76, S/dataset.cpp:39-247
 */
#include "lamm_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char* lor_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- RNG --- */
/* std::mt19937_64 (its sequence is fixed by the C++ standard) plus the
 * reference's hand-coded draws, H/rng.hpp:25-81. */
typedef struct {
    uint64_t mt[312];
    int mti;
    double spare;
    int have_spare;
} Rng;

static void rng_init(Rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
    r->spare = 0.0;
    r->have_spare = 0;
}

static uint64_t rng_u64(Rng* r) {
    if (r->mti >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->mti = 0;
    }
    uint64_t y = r->mt[r->mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

static double rng_uniform(Rng* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }
static double rng_uniform_in(Rng* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }

static double rng_normal(Rng* r) { /* H/rng.hpp:37-49 */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = 1.0 - rng_uniform(r);
    const double u2 = rng_uniform(r);
    const double rr = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rr * sin(theta);
    r->have_spare = 1;
    return rr * cos(theta);
}
static double rng_normal_ms(Rng* r, double mean, double sd) { return mean + sd * rng_normal(r); }

static uint64_t rng_bounded(Rng* r, uint64_t n) { /* H/rng.hpp:54-60 */
    if (n == 0) return 0;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x = rng_u64(r);
    while (x >= limit) x = rng_u64(r);
    return x % n;
}

uint64_t lor_mix_seed(uint64_t a, uint64_t b) { /* H/rng.hpp:18-23 */
    uint64_t z = a + 0x9e3779b97f4a7c15ULL + b * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static void rng_permutation(Rng* r, int64_t n, int64_t* p) { /* H/rng.hpp:63-75 */
    for (int64_t k = 0; k < n; ++k) p[k] = k;
    for (int64_t k = n; k > 1; --k) {
        const int64_t j = (int64_t)rng_bounded(r, (uint64_t)k);
        const int64_t t = p[k - 1];
        p[k - 1] = p[j];
        p[j] = t;
    }
}

void lor_rng_normals(uint64_t seed, int64_t n, double* out) {
    Rng r;
    rng_init(&r, seed);
    for (int64_t k = 0; k < n; ++k) out[k] = rng_normal(&r);
}
void lor_rng_uniforms(uint64_t seed, int64_t n, double* out) {
    Rng r;
    rng_init(&r, seed);
    for (int64_t k = 0; k < n; ++k) out[k] = rng_uniform(&r);
}
void lor_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
    Rng r;
    rng_init(&r, seed);
    for (int64_t k = 0; k < n; ++k) out[k] = rng_u64(&r);
}
void lor_rng_bounded(uint64_t seed, int64_t n, uint64_t bound, uint64_t* out) {
    Rng r;
    rng_init(&r, seed);
    for (int64_t k = 0; k < n; ++k) out[k] = rng_bounded(&r, bound);
}
void lor_rng_permutation(uint64_t seed, int64_t n, int64_t* out) {
    Rng r;
    rng_init(&r, seed);
    rng_permutation(&r, n, out);
}

/* ------------------------------------------------------ neighbour list --- */
typedef struct {
    int64_t n;
    int32_t *i, *j;
    double *dist, *unit;
} Pairs;

static int validate_system(int32_t n, const double* pos, const int32_t* Z) { /* S/core.cpp:10-20 */
    if (n < 1) return set_err("system has no atoms"), 1;
    for (int64_t k = 0; k < 3 * (int64_t)n; ++k)
        if (!isfinite(pos[k])) return set_err("non-finite coordinate"), 1;
    for (int32_t a = 0; a < n; ++a)
        if (Z[a] < 1 || Z[a] > 118) return set_err("atomic number outside [1, 118]"), 1;
    return 0;
}

/* Periodic cells (SURVEY.md §8(f) extension; the reference has none, so this is
 * parity-unpinned): sample s is periodic when g_cells holds a nonzero 3x3 cell
 * (rows = lattice vectors) for it, with per-axis periodicity g_pbc[s][k] (NULL:
 * all three axes periodic). A pair is (i, j, n): atom j's image shifted by the
 * integer vector n relative to its minimum image,
 *   f_k = sum_c d_c cinv[c][k];  f_k -= rint(f_k) on periodic axes;
 *   g_k = f_k - n_k;  d_c = sum_k g_k cell[k][c]         (d = p_i - p_j, left to right,
 * no contraction; the device kernels use the same sequence with __d*_rn), with
 * n_k in [-m_k, m_k], m_k = floor(0.5 + cutoff * b_k (1 + 1e-9)) on periodic axes
 * (b_k = |column k of cinv| = 1 / perpendicular width k) and 0 otherwise: every
 * image within the cutoff (|f_k| < cutoff b_k for |d| < cutoff, |f_k - rint| <= 1/2).
 * Order: i-major, j ascending, then n lexicographic; (i, i, 0) excluded. Cells at
 * least 2 * cutoff wide on every periodic axis give m = 0: the minimum image. */
static _Thread_local const double* g_cells = NULL;
static _Thread_local const double* g_cellinv = NULL;
static _Thread_local const uint8_t* g_pbc = NULL;

/* 3x3 inverse by cofactors (rows = lattice vectors), the same expression
 * sequence as the device library's cell_inverse (device.cuh); 1 if singular. */
int lor_cell_inverse(const double* m, double* inv) {
    const double c00 = m[4] * m[8] - m[5] * m[7], c01 = m[5] * m[6] - m[3] * m[8], c02 = m[3] * m[7] - m[4] * m[6];
    const double c10 = m[2] * m[7] - m[1] * m[8], c11 = m[0] * m[8] - m[2] * m[6], c12 = m[1] * m[6] - m[0] * m[7];
    const double c20 = m[1] * m[5] - m[2] * m[4], c21 = m[2] * m[3] - m[0] * m[5], c22 = m[0] * m[4] - m[1] * m[3];
    const double det = (m[0] * c00 + m[1] * c01) + m[2] * c02;
    if (!(det != 0.0)) return set_err("cell: singular"), 1;
    const double cof[9] = {c00, c10, c20, c01, c11, c21, c02, c12, c22};
    for (int k = 0; k < 9; ++k) inv[k] = cof[k] / det;
    return 0;
}

void lor_set_cells(const double* cells, const double* cellinv) {
    g_cells = cells;
    g_cellinv = cellinv;
}

void lor_set_pbc(const uint8_t* pbc) { g_pbc = pbc; }

/* Image range per axis (-1: non-periodic axis of a periodic sample). */
void lor_image_range(const double* ci, const uint8_t* pbc, double cutoff, int* m) {
    for (int k = 0; k < 3; ++k) {
        if (pbc && !pbc[k]) {
            m[k] = -1;
            continue;
        }
        const double b = sqrt((ci[k] * ci[k] + ci[3 + k] * ci[3 + k]) + ci[6 + k] * ci[6 + k]);
        m[k] = (int)floor(0.5 + cutoff * b * (1.0 + 1e-9));
    }
}

static const double* cell_of(int64_t s) {
    if (!g_cells) return NULL;
    const double* c = g_cells + 9 * s;
    for (int k = 0; k < 9; ++k)
        if (c[k] != 0.0) return c;
    return NULL;
}

static void image_disp(const double* cell, const double* ci, const int* m, const int* n, double* d0, double* d1,
                       double* d2) {
    double f[3];
    for (int k = 0; k < 3; ++k) {
        const double a = *d0 * ci[k], b = *d1 * ci[3 + k], c = *d2 * ci[6 + k];
        f[k] = (a + b) + c;
        if (m[k] >= 0) f[k] = f[k] - rint(f[k]);
        f[k] = f[k] - (double)n[k];
    }
    double o[3];
    for (int c = 0; c < 3; ++c) {
        const double a = f[0] * cell[c], b = f[1] * cell[3 + c], e = f[2] * cell[6 + c];
        o[c] = (a + b) + e;
    }
    *d0 = o[0], *d1 = o[1], *d2 = o[2];
}

/* S/core.cpp:30-48: all ordered pairs, r < cutoff strictly, i-major, j-ascending.
 * cell/ci non-NULL: the image pairs of a periodic sample (pbc: its per-axis flags,
 * NULL = all periodic), see above. */
static int build_pairs_cell(int32_t n, const double* pos, const int32_t* Z, double cutoff, const double* cell,
                            const double* ci, const uint8_t* pbc, Pairs* out);
static int build_pairs_cell(int32_t n, const double* pos, const int32_t* Z, double cutoff, const double* cell,
                            const double* ci, const uint8_t* pbc, Pairs* out) {
    if (validate_system(n, pos, Z)) return 1;
    if (!(cutoff > 0.0)) return set_err("cutoff must be positive"), 1;
    int64_t cap = 64, cnt = 0;
    out->i = malloc(sizeof(int32_t) * cap);
    out->j = malloc(sizeof(int32_t) * cap);
    out->dist = malloc(sizeof(double) * cap);
    out->unit = malloc(sizeof(double) * 3 * cap);
    int m[3] = {0, 0, 0};
    if (cell) lor_image_range(ci, pbc, cutoff, m);
    const int w0 = 2 * (m[0] > 0 ? m[0] : 0) + 1, w1 = 2 * (m[1] > 0 ? m[1] : 0) + 1,
              w2 = 2 * (m[2] > 0 ? m[2] : 0) + 1;
    const int nimg = w0 * w1 * w2;
    for (int32_t i = 0; i < n; ++i) {
        for (int32_t j = 0; j < n; ++j) for (int img = 0; img < nimg; ++img) {
            const int sh[3] = {img / (w1 * w2) - (w0 - 1) / 2, (img / w2) % w1 - (w1 - 1) / 2, img % w2 - (w2 - 1) / 2};
            if (j == i && sh[0] == 0 && sh[1] == 0 && sh[2] == 0) continue;
            double d0 = pos[3 * i] - pos[3 * j], d1 = pos[3 * i + 1] - pos[3 * j + 1], d2 = pos[3 * i + 2] - pos[3 * j + 2];
            if (cell) image_disp(cell, ci, m, sh, &d0, &d1, &d2);
            const double r = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            if (r < cutoff) {
                if (cnt == cap) {
                    cap *= 2;
                    out->i = realloc(out->i, sizeof(int32_t) * cap);
                    out->j = realloc(out->j, sizeof(int32_t) * cap);
                    out->dist = realloc(out->dist, sizeof(double) * cap);
                    out->unit = realloc(out->unit, sizeof(double) * 3 * cap);
                }
                const double s = 1.0 / r;
                out->i[cnt] = i;
                out->j[cnt] = j;
                out->dist[cnt] = r;
                out->unit[3 * cnt] = s * d0;
                out->unit[3 * cnt + 1] = s * d1;
                out->unit[3 * cnt + 2] = s * d2;
                ++cnt;
            }
        }
    }
    out->n = cnt;
    return 0;
}

static void free_pairs(Pairs* p) {
    free(p->i);
    free(p->j);
    free(p->dist);
    free(p->unit);
}

int64_t lor_neighbor_list(int32_t n, const double* pos, const int32_t* Z, double cutoff, int64_t cap, int32_t* oi,
                          int32_t* oj, double* odist, double* ounit) {
    Pairs p;
    const double* cell = cell_of(0);
    if (build_pairs_cell(n, pos, Z, cutoff, cell, cell ? g_cellinv : NULL, g_pbc, &p)) return -1;
    for (int64_t k = 0; k < p.n && k < cap; ++k) {
        oi[k] = p.i[k];
        oj[k] = p.j[k];
        odist[k] = p.dist[k];
        for (int c = 0; c < 3; ++c) ounit[3 * k + c] = p.unit[3 * k + c];
    }
    const int64_t cnt = p.n;
    free_pairs(&p);
    return cnt;
}

/* --------------------------------------------------------------- model --- */
/* Parameter views over the flat for_each_tensor layout (H/model.hpp:46-66). */
typedef struct {
    int H, L, K, D;
    double rc;
    double* emb;    /* 118 x H */
    double** filt;  /* L of H x K */
    double** upd;   /* L of H x H */
    double* ehead;  /* H x D */
    double* fhead;  /* (2H+K) x D */
} Params;

int64_t lor_param_count(int H, int L, int K, int D) {
    return 118LL * H + (int64_t)L * H * K + (int64_t)L * H * H + (int64_t)H * D + (int64_t)(2 * H + K) * D;
}

static void params_view(Params* p, int H, int L, int K, double rc, int D, double* flat) {
    p->H = H, p->L = L, p->K = K, p->D = D, p->rc = rc;
    p->filt = malloc(sizeof(double*) * (L > 0 ? L : 1));
    p->upd = malloc(sizeof(double*) * (L > 0 ? L : 1));
    double* q = flat;
    p->emb = q, q += 118 * H;
    for (int l = 0; l < L; ++l) p->filt[l] = q, q += H * K;
    for (int l = 0; l < L; ++l) p->upd[l] = q, q += H * H;
    p->ehead = q, q += H * D;
    p->fhead = q;
}
static void params_free(Params* p) {
    free(p->filt);
    free(p->upd);
}

static int validate_config(int H, int L, int K, double rc, int D) { /* S/model.cpp:115-121 */
    if (H < 1) return set_err("model: hidden must be >= 1"), 1;
    if (L < 0) return set_err("model: layers must be >= 0"), 1;
    if (K < 2) return set_err("model: rbf must be >= 2"), 1;
    if (!(rc > 0.0)) return set_err("model: cutoff must be positive"), 1;
    if (D < 1) return set_err("model: heads must be >= 1"), 1;
    return 0;
}

int lor_init_params(int H, int L, int K, double rc, int D, uint64_t seed, double* out) {
    if (validate_config(H, L, K, rc, D)) return 1;
    Rng r;
    rng_init(&r, seed);
    const int64_t total = lor_param_count(H, L, K, D);
    int64_t o = 0;
    /* S/model.cpp:177-193 + init_heads :163-171: tensor order, U(+-scale) */
    for (int64_t k = 0; k < 118LL * H; ++k) out[o++] = rng_uniform_in(&r, -1.0, 1.0);
    const double sf = 1.0 / sqrt((double)K), su = 1.0 / sqrt((double)H);
    for (int l = 0; l < L; ++l)
        for (int64_t k = 0; k < (int64_t)H * K; ++k) out[o++] = rng_uniform_in(&r, -sf, sf);
    for (int l = 0; l < L; ++l)
        for (int64_t k = 0; k < (int64_t)H * H; ++k) out[o++] = rng_uniform_in(&r, -su, su);
    for (int64_t k = 0; k < (int64_t)H * D; ++k) out[o++] = rng_uniform_in(&r, -su, su);
    const double sh = 1.0 / sqrt((double)(2 * H + K));
    for (int64_t k = 0; k < (int64_t)(2 * H + K) * D; ++k) out[o++] = rng_uniform_in(&r, -sh, sh);
    return o == total ? 0 : 2;
}

static const double kPi = 3.14159265358979323846;

/* ForwardCache (H/model.hpp:86-95) */
typedef struct {
    int n;
    Pairs pr;
    double* fc;   /* P */
    double* rbf;  /* P x K */
    double* h;    /* (L+1) x n x H */
    double* mt;   /* L x n x H */
    const int32_t* Z;
} Cache;

static int run_encoder_s(const Params* p, int32_t n, const double* pos, const int32_t* Z, int64_t s, Cache* c);
static int run_encoder(const Params* p, int32_t n, const double* pos, const int32_t* Z, Cache* c) {
    return run_encoder_s(p, n, pos, Z, 0, c);
}
/* s: the sample's index for its (optional) cell */
static int run_encoder_s(const Params* p, int32_t n, const double* pos, const int32_t* Z, int64_t s, Cache* c) {
    /* S/model.cpp:37-110 */
    const int H = p->H, K = p->K, L = p->L;
    const double* cell = cell_of(s);
    if (build_pairs_cell(n, pos, Z, p->rc, cell, cell ? g_cellinv + 9 * s : NULL, g_pbc ? g_pbc + 3 * s : NULL,
                         &c->pr))
        return 1;
    const int64_t P = c->pr.n;
    c->n = n;
    c->Z = Z;
    c->fc = malloc(sizeof(double) * (P ? P : 1));
    c->rbf = malloc(sizeof(double) * (P ? P : 1) * K);
    const double width = p->rc / (double)(K - 1);
    const double inv = 1.0 / (2.0 * width * width);
    for (int64_t q = 0; q < P; ++q) {
        const double r = c->pr.dist[q];
        for (int k = 0; k < K; ++k) {
            const double d = r - width * (double)k;
            c->rbf[q * K + k] = exp(-d * d * inv);
        }
        c->fc[q] = 0.5 * (cos(kPi * r / p->rc) + 1.0);
    }
    c->h = calloc((size_t)(L + 1) * n * H, sizeof(double));
    c->mt = calloc((size_t)(L > 0 ? L : 1) * n * H, sizeof(double));
    for (int32_t i = 0; i < n; ++i)
        for (int a = 0; a < H; ++a) c->h[(int64_t)i * H + a] = p->emb[(int64_t)(Z[i] - 1) * H + a];
    double* t = malloc(sizeof(double) * n * H);
    double* msg = malloc(sizeof(double) * n * H);
    double* filt = malloc(sizeof(double) * H);
    for (int l = 0; l < L; ++l) {
        const double* h = c->h + (int64_t)l * n * H;
        double* hn = c->h + (int64_t)(l + 1) * n * H;
        double* mt = c->mt + (int64_t)l * n * H;
        const double* wf = p->filt[l];
        const double* wu = p->upd[l];
        for (int64_t k = 0; k < (int64_t)n * H; ++k) t[k] = tanh(h[k]);
        memset(msg, 0, sizeof(double) * n * H);
        for (int64_t q = 0; q < P; ++q) {
            const double* rb = c->rbf + q * K;
            for (int a = 0; a < H; ++a) {
                double acc = 0.0;
                for (int k = 0; k < K; ++k) acc += wf[a * K + k] * rb[k];
                filt[a] = acc * c->fc[q];
            }
            const int64_t i = c->pr.i[q], j = c->pr.j[q];
            for (int a = 0; a < H; ++a) msg[i * H + a] += t[j * H + a] * filt[a];
        }
        for (int64_t k = 0; k < (int64_t)n * H; ++k) mt[k] = tanh(msg[k]);
        for (int32_t i = 0; i < n; ++i)
            for (int b = 0; b < H; ++b) {
                double acc = h[(int64_t)i * H + b];
                for (int a = 0; a < H; ++a) acc += wu[b * H + a] * mt[(int64_t)i * H + a];
                hn[(int64_t)i * H + b] = acc;
            }
    }
    free(t);
    free(msg);
    free(filt);
    return 0;
}

static void cache_free(Cache* c) {
    free_pairs(&c->pr);
    free(c->fc);
    free(c->rbf);
    free(c->h);
    free(c->mt);
}

/* predict_energy S/model.cpp:208-218 + force_kernel :223-253 */
static void heads_forward(const Params* p, const Cache* c, double* energy, double* forces) {
    const int H = p->H, K = p->K, D = p->D;
    const int n = c->n;
    const double* hl = c->h + (int64_t)p->L * n * H;
    for (int d = 0; d < D; ++d) energy[d] = 0.0;
    for (int32_t i = 0; i < n; ++i)
        for (int a = 0; a < H; ++a)
            for (int d = 0; d < D; ++d) energy[d] += p->ehead[a * D + d] * hl[(int64_t)i * H + a];
    double* t = malloc(sizeof(double) * n * H);
    for (int64_t k = 0; k < (int64_t)n * H; ++k) t[k] = tanh(hl[k]);
    memset(forces, 0, sizeof(double) * D * n * 3);
    double* w = malloc(sizeof(double) * D);
    for (int64_t q = 0; q < c->pr.n; ++q) {
        const int64_t i = c->pr.i[q], j = c->pr.j[q];
        const double* rb = c->rbf + q * K;
        for (int d = 0; d < D; ++d) {
            double acc = 0.0;
            for (int a = 0; a < H; ++a) {
                acc += p->fhead[a * D + d] * (t[i * H + a] + t[j * H + a]);
                acc += p->fhead[(H + a) * D + d] * (t[i * H + a] * t[j * H + a]);
            }
            for (int k = 0; k < K; ++k) acc += p->fhead[(2 * H + k) * D + d] * rb[k];
            w[d] = acc;
        }
        for (int d = 0; d < D; ++d)
            for (int cc = 0; cc < 3; ++cc)
                forces[((int64_t)d * n + i) * 3 + cc] += w[d] * c->fc[q] * c->pr.unit[3 * q + cc];
    }
    free(w);
    free(t);
}

int lor_forward(int H, int L, int K, double rc, int D, const double* params, int32_t B, const int64_t* atom_ptr,
                const double* pos, const int32_t* Z, double* out_energy, double* out_forces) {
    if (validate_config(H, L, K, rc, D)) return 1;
    Params p;
    params_view(&p, H, L, K, rc, D, (double*)params);
    int st = 0;
    for (int s = 0; s < B && !st; ++s) {
        Cache c;
        const int32_t n = (int32_t)(atom_ptr[s + 1] - atom_ptr[s]);
        st = run_encoder_s(&p, n, pos + 3 * atom_ptr[s], Z + atom_ptr[s], s, &c);
        if (st) break;
        heads_forward(&p, &c, out_energy + (int64_t)s * D, out_forces + 3 * D * atom_ptr[s]);
        cache_free(&c);
    }
    params_free(&p);
    return st;
}

int lor_forward_cache(int H, int L, int K, double rc, int D, const double* params, int32_t n, const double* pos,
                      const int32_t* Z, double* h_all, double* mt_all) {
    if (validate_config(H, L, K, rc, D)) return 1;
    Params p;
    params_view(&p, H, L, K, rc, D, (double*)params);
    Cache c;
    const int st = run_encoder(&p, n, pos, Z, &c);
    if (!st) {
        memcpy(h_all, c.h, sizeof(double) * (L + 1) * n * H);
        if (L > 0) memcpy(mt_all, c.mt, sizeof(double) * L * n * H);
        cache_free(&c);
    }
    params_free(&p);
    return st;
}

/* model::backward, S/model.cpp:299-425; grads accumulated (+=) */
static void backward_one(const Params* p, const Cache* c, const double* up_e, const double* up_f, Params* g) {
    const int H = p->H, K = p->K, D = p->D, L = p->L;
    const int n = c->n;
    const int64_t P = c->pr.n;
    const int64_t NH = (int64_t)n * H;
    const double* hl = c->h + (int64_t)L * NH;
    double* tl = malloc(sizeof(double) * NH);
    for (int64_t k = 0; k < NH; ++k) tl[k] = tanh(hl[k]);
    double* gh = calloc((size_t)NH, sizeof(double));
    double* gt = calloc((size_t)NH, sizeof(double));
    for (int d = 0; d < D; ++d) {
        const double ge = up_e[d];
        if (ge == 0.0) continue;
        for (int32_t i = 0; i < n; ++i)
            for (int a = 0; a < H; ++a) {
                g->ehead[a * D + d] += hl[(int64_t)i * H + a] * ge;
                gh[(int64_t)i * H + a] += p->ehead[a * D + d] * ge;
            }
    }
    const int Q = 2 * H + K;
    double* gw = malloc(sizeof(double) * D);
    double* gphi = malloc(sizeof(double) * Q);
    for (int64_t q = 0; q < P; ++q) {
        const int64_t i = c->pr.i[q], j = c->pr.j[q];
        const double env = c->fc[q];
        int any = 0;
        for (int d = 0; d < D; ++d) {
            double acc = 0.0;
            for (int cc = 0; cc < 3; ++cc) acc += up_f[((int64_t)d * n + i) * 3 + cc] * c->pr.unit[3 * q + cc];
            gw[d] = env * acc;
            any = any || gw[d] != 0.0;
        }
        if (!any) continue;
        const double* rb = c->rbf + q * K;
        for (int qq = 0; qq < Q; ++qq) {
            double phi;
            if (qq < H) phi = tl[i * H + qq] + tl[j * H + qq];
            else if (qq < 2 * H) phi = tl[i * H + qq - H] * tl[j * H + qq - H];
            else phi = rb[qq - 2 * H];
            double gg = 0.0;
            for (int d = 0; d < D; ++d) {
                g->fhead[qq * D + d] += phi * gw[d];
                gg += p->fhead[qq * D + d] * gw[d];
            }
            gphi[qq] = gg;
        }
        for (int a = 0; a < H; ++a) {
            gt[i * H + a] += gphi[a] + gphi[H + a] * tl[j * H + a];
            gt[j * H + a] += gphi[a] + gphi[H + a] * tl[i * H + a];
        }
    }
    for (int64_t k = 0; k < NH; ++k) gh[k] += gt[k] * (1.0 - tl[k] * tl[k]);

    double* filt = malloc(sizeof(double) * H);
    double* gpsi = malloc(sizeof(double) * H);
    double* gm = malloc(sizeof(double) * NH);
    double* tll = malloc(sizeof(double) * NH);
    double* gtl = malloc(sizeof(double) * NH);
    for (int l = L - 1; l >= 0; --l) {
        const double* mt = c->mt + (int64_t)l * NH;
        const double* wu = p->upd[l];
        const double* wf = p->filt[l];
        memset(gm, 0, sizeof(double) * NH);
        for (int32_t i = 0; i < n; ++i)
            for (int b = 0; b < H; ++b) {
                const double gg = gh[(int64_t)i * H + b];
                if (gg == 0.0) continue;
                for (int a = 0; a < H; ++a) {
                    g->upd[l][b * H + a] += gg * mt[(int64_t)i * H + a];
                    gm[(int64_t)i * H + a] += wu[b * H + a] * gg;
                }
            }
        for (int64_t k = 0; k < NH; ++k) gm[k] *= 1.0 - mt[k] * mt[k];
        const double* hl_ = c->h + (int64_t)l * NH;
        for (int64_t k = 0; k < NH; ++k) tll[k] = tanh(hl_[k]);
        memset(gtl, 0, sizeof(double) * NH);
        for (int64_t q = 0; q < P; ++q) {
            const int64_t i = c->pr.i[q], j = c->pr.j[q];
            const double env = c->fc[q];
            const double* rb = c->rbf + q * K;
            for (int a = 0; a < H; ++a) {
                double acc = 0.0;
                for (int k = 0; k < K; ++k) acc += wf[a * K + k] * rb[k];
                filt[a] = acc * env;
            }
            for (int a = 0; a < H; ++a) {
                const double gg = gm[i * H + a];
                if (gg == 0.0) continue;
                gtl[j * H + a] += gg * filt[a];
                gpsi[a] = gg * tll[j * H + a] * env;
                for (int k = 0; k < K; ++k) g->filt[l][a * K + k] += gpsi[a] * rb[k];
            }
        }
        for (int64_t k = 0; k < NH; ++k) gh[k] += gtl[k] * (1.0 - tll[k] * tll[k]);
    }
    for (int32_t i = 0; i < n; ++i) {
        const int64_t z = c->Z[i] - 1;
        for (int a = 0; a < H; ++a) g->emb[z * H + a] += gh[(int64_t)i * H + a];
    }
    free(filt);
    free(gpsi);
    free(gm);
    free(tll);
    free(gtl);
    free(gw);
    free(gphi);
    free(gh);
    free(gt);
    free(tl);
}

int lor_backward(int H, int L, int K, double rc, int D, const double* params, int32_t B, const int64_t* atom_ptr,
                 const double* pos, const int32_t* Z, const double* up_energy, const double* up_forces,
                 double* grads_accum) {
    if (validate_config(H, L, K, rc, D)) return 1;
    Params p, g;
    params_view(&p, H, L, K, rc, D, (double*)params);
    params_view(&g, H, L, K, rc, D, grads_accum);
    int st = 0;
    for (int s = 0; s < B; ++s) {
        Cache c;
        const int32_t n = (int32_t)(atom_ptr[s + 1] - atom_ptr[s]);
        st = run_encoder_s(&p, n, pos + 3 * atom_ptr[s], Z + atom_ptr[s], s, &c);
        if (st) break;
        backward_one(&p, &c, up_energy + (int64_t)s * D, up_forces + 3 * D * atom_ptr[s], &g);
        cache_free(&c);
    }
    params_free(&p);
    params_free(&g);
    return st;
}

/* ---------------------------------------------------------------- loss --- */
/* normalize_labels S/loss.cpp:113-126 for one sample; table rows are dense in Z
 * with presence flags standing in for the std::map. */
static int normalize_one(int32_t n, const int32_t* Z, int ds, int em, int fm, double energy, const double* forces,
                         int ntab, const double* rho, const uint8_t* rho_has, const double* mean, const double* stdv,
                         const double* fstd, const uint8_t* has, double* oe, double* of) {
    if (ds < 0 || ds >= ntab) return set_err("dataset index outside reference table"), 1;
    *oe = 0.0;
    if (em) {
        if (!has[ds]) return set_err("normalize_labels: dataset has no fitted energy statistics"), 1;
        double total = 0.0;
        for (int32_t a = 0; a < n; ++a)
            if (rho_has[ds * 119 + Z[a]]) total += rho[ds * 119 + Z[a]];
        *oe = (energy - total - mean[ds]) / stdv[ds];
    }
    const double s = 1.0 / fstd[ds];
    for (int64_t k = 0; k < 3 * (int64_t)n; ++k) of[k] = fm ? s * forces[k] : 0.0;
    return 0;
}

int lor_normalize_labels(int32_t B, const int64_t* atom_ptr, const double* pos, const int32_t* Z, const int32_t* dsidx,
                         const uint8_t* emask, const uint8_t* fmask, const double* energy, const double* forces,
                         int ntab, const double* rho, const uint8_t* rho_has, const double* mean, const double* stdv,
                         const double* fstd, const uint8_t* has, double* out_energy, double* out_forces) {
    (void)pos;
    for (int s = 0; s < B; ++s) {
        const int64_t o = atom_ptr[s];
        if (normalize_one((int32_t)(atom_ptr[s + 1] - o), Z + o, dsidx[s], emask[s], fmask[s], energy[s],
                          forces + 3 * o, ntab, rho, rho_has, mean, stdv, fstd, has, out_energy + s,
                          out_forces + 3 * o))
            return 1;
    }
    return 0;
}

/* masked_loss_impl, S/loss.cpp:140-213 (Eq. 5). */
int lor_loss_grad(int32_t B, const int64_t* atom_ptr, int D, const int32_t* dsidx, const uint8_t* emask,
                  const uint8_t* fmask, const double* energy, const double* forces, const double* pred_energy,
                  const double* pred_forces, double lambda_e, double lambda_f, double* breakdown, double* g_energy,
                  double* g_forces) {
    if (!(lambda_e >= 0.0) || !(lambda_f >= 0.0)) return set_err("masked_loss: lambdas must be non-negative"), 1;
    int me = 0, mf = 0;
    for (int s = 0; s < B; ++s) {
        if (dsidx[s] < 0) return set_err("negative dataset index"), 1;
        if (dsidx[s] >= D) return set_err("masked_loss: dataset index outside prediction heads"), 1;
        me += emask[s] != 0;
        mf += fmask[s] != 0;
    }
    if (g_energy) memset(g_energy, 0, sizeof(double) * B * D);
    if (g_forces) memset(g_forces, 0, sizeof(double) * 3 * D * atom_ptr[B]);
    const double we = me > 0 ? lambda_e / (double)me : 0.0;
    const double wf = mf > 0 ? lambda_f / (double)mf : 0.0;
    double eterm = 0.0, fterm = 0.0;
    for (int s = 0; s < B; ++s) {
        const int64_t d = dsidx[s];
        const int64_t n = atom_ptr[s + 1] - atom_ptr[s];
        const double* pf = pred_forces + 3 * D * atom_ptr[s];
        if (emask[s]) {
            const double diff = pred_energy[(int64_t)s * D + d] - energy[s];
            eterm += we * fabs(diff);
            if (g_energy && diff != 0.0) g_energy[(int64_t)s * D + d] = diff > 0.0 ? we : -we;
        }
        if (fmask[s]) {
            const double ws = wf / (double)n;
            for (int64_t j = 0; j < n; ++j) {
                double sq = 0.0, diff[3];
                for (int c = 0; c < 3; ++c) {
                    diff[c] = pf[(d * n + j) * 3 + c] - forces[3 * (atom_ptr[s] + j) + c];
                    sq += diff[c] * diff[c];
                }
                const double dist = sqrt(sq);
                fterm += ws * dist;
                if (g_forces && dist > 0.0)
                    for (int c = 0; c < 3; ++c) g_forces[3 * D * atom_ptr[s] + (d * n + j) * 3 + c] = ws * diff[c] / dist;
            }
        }
    }
    breakdown[0] = eterm + fterm;
    breakdown[1] = eterm;
    breakdown[2] = fterm;
    breakdown[3] = me;
    breakdown[4] = mf;
    breakdown[5] = me == 0;
    breakdown[6] = mf == 0;
    return 0;
}

/* ------------------------------------------------------------- denoise --- */
int lor_apply_displacements(int32_t n, const double* pos, const int32_t* Z, const double* deltas, int scheme,
                            double* noisy, double* labels) { /* S/denoise.cpp:7-29 */
    if (validate_system(n, pos, Z)) return 1;
    double m0 = 0.0, m1 = 0.0, m2 = 0.0;
    if (scheme) {
        for (int32_t a = 0; a < n; ++a) {
            m0 = m0 + deltas[3 * a];
            m1 = m1 + deltas[3 * a + 1];
            m2 = m2 + deltas[3 * a + 2];
        }
        const double s = 1.0 / (double)n;
        m0 = s * m0, m1 = s * m1, m2 = s * m2;
    }
    const double m[3] = {m0, m1, m2};
    for (int32_t a = 0; a < n; ++a)
        for (int c = 0; c < 3; ++c) {
            const double e = scheme ? deltas[3 * a + c] - m[c] : deltas[3 * a + c];
            noisy[3 * a + c] = pos[3 * a + c] + e;
            labels[3 * a + c] = -1.0 * e;
        }
    return 0;
}

int lor_apply_noise(int32_t n, const double* pos, const int32_t* Z, double sigma, int scheme, uint64_t seed,
                    double* noisy, double* labels) { /* S/denoise.cpp:31-40 */
    if (!(sigma > 0.0)) return set_err("apply_noise: sigma must be positive"), 1;
    Rng r;
    rng_init(&r, seed);
    double* d = malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
    for (int64_t k = 0; k < 3 * (int64_t)n; ++k) d[k] = rng_normal_ms(&r, 0.0, sigma);
    const int st = lor_apply_displacements(n, pos, Z, d, scheme, noisy, labels);
    free(d);
    return st;
}

/* ---------------------------------------------------------- train step --- */
/* One simulated worker of the step body (S/trainer.cpp:262-292): denoise,
 * normalize, forward, per-worker masked_loss_grad and backward accumulated
 * into g; returns the worker's loss in *loss_out. */
static int worker_body(const Params* pp, Params* gg, int gi, int B, int D, const int64_t* atom_ptr,
                       const double* pos, const int32_t* Z, const int32_t* dsidx, const uint8_t* emask,
                       const uint8_t* fmask, const double* energy, const double* forces,
                       const uint8_t* denoise_flag, int ntab, const double* rho, const uint8_t* rho_has,
                       const double* mean, const double* stdv, const double* fstd, const uint8_t* has,
                       double noise_sigma, int noise_scheme, uint64_t seed, int64_t step, double lambda_e,
                       double lambda_f, double* loss_out) {
    const Params p = *pp;
    const uint64_t kNoiseTag = 0x4e4f4953;
    int st = 0;
    *loss_out = 0.0;
    const int64_t base = atom_ptr[(int64_t)gi * B];
    const int64_t natoms = atom_ptr[(int64_t)(gi + 1) * B] - base;
    int64_t* lptr = malloc(sizeof(int64_t) * (B + 1));
    for (int b = 0; b <= B; ++b) lptr[b] = atom_ptr[(int64_t)gi * B + b] - base;
    double* xs = malloc(sizeof(double) * 3 * natoms);
    double* le = malloc(sizeof(double) * B);
    double* lf = malloc(sizeof(double) * 3 * natoms);
    int32_t* ld = malloc(sizeof(int32_t) * B);
    uint8_t* lem = malloc(B);
    uint8_t* lfm = malloc(B);
    double* pe = malloc(sizeof(double) * B * D);
    double* pf = malloc(sizeof(double) * 3 * D * natoms);
    double* ge = malloc(sizeof(double) * B * D);
    double* gf = malloc(sizeof(double) * 3 * D * natoms);
    Cache* caches = calloc((size_t)B, sizeof(Cache));
    for (int b = 0; b < B && !st; ++b) {
        const int pos_ = gi * B + b;
        const int64_t o = atom_ptr[pos_], lo = lptr[b];
        const int32_t n = (int32_t)(atom_ptr[pos_ + 1] - o);
        ld[b] = dsidx[pos_];
        if (denoise_flag && denoise_flag[pos_]) { /* make_denoising_sample S/denoise.cpp:42-53 */
            const uint64_t ns = lor_mix_seed(lor_mix_seed(seed, kNoiseTag + (uint64_t)step), (uint64_t)pos_);
            double* lab = malloc(sizeof(double) * 3 * n);
            st = lor_apply_noise(n, pos + 3 * o, Z + o, noise_sigma, noise_scheme, ns, xs + 3 * lo, lab);
            lem[b] = 0, lfm[b] = 1;
            if (!st)
                st = normalize_one(n, Z + o, ld[b], 0, 1, 0.0, lab, ntab, rho, rho_has, mean, stdv, fstd, has,
                                   le + b, lf + 3 * lo);
            free(lab);
        } else {
            memcpy(xs + 3 * lo, pos + 3 * o, sizeof(double) * 3 * n);
            lem[b] = emask[pos_], lfm[b] = fmask[pos_];
            st = normalize_one(n, Z + o, ld[b], lem[b], lfm[b], energy[pos_], forces + 3 * o, ntab, rho, rho_has,
                               mean, stdv, fstd, has, le + b, lf + 3 * lo);
        }
        if (!st) st = run_encoder_s(&p, n, xs + 3 * lo, Z + o, pos_, &caches[b]);
        if (!st) heads_forward(&p, &caches[b], pe + (int64_t)b * D, pf + 3 * D * lo);
    }
    double bd[7];
    if (!st)
        st = lor_loss_grad(B, lptr, D, ld, lem, lfm, le, lf, pe, pf, lambda_e, lambda_f, bd, ge, gf);
    if (!st) {
        *loss_out = bd[0];
        for (int b = 0; b < B; ++b)
            backward_one(&p, &caches[b], ge + (int64_t)b * D, gf + 3 * D * lptr[b], gg);
    }
    for (int b = 0; b < B; ++b)
        if (caches[b].h) cache_free(&caches[b]);
    free(caches);
    free(lptr), free(xs), free(le), free(lf), free(ld), free(lem), free(lfm);
    free(pe), free(pf), free(ge), free(gf);
    return st;
}


int lor_train_step(int H, int L, int K, double rc, int D, int G, int B, const int64_t* atom_ptr, const double* pos,
                   const int32_t* Z, const int32_t* dsidx, const uint8_t* emask, const uint8_t* fmask,
                   const double* energy, const double* forces, const uint8_t* denoise_flag, int ntab,
                   const double* rho, const uint8_t* rho_has, const double* mean, const double* stdv,
                   const double* fstd, const uint8_t* has, double noise_sigma, int noise_scheme, uint64_t seed,
                   int64_t step, double lambda_e, double lambda_f, double lr, double clip, double decay, double eps,
                   double* params, double* rms_v, double* out_loss, double* out_grad_norm, double* out_grads) {
    /* S/trainer.cpp:258-327 */
    if (validate_config(H, L, K, rc, D)) return 1;
    const int64_t NP = lor_param_count(H, L, K, D);
    double* grads = calloc((size_t)NP, sizeof(double));
    Params p, g;
    params_view(&p, H, L, K, rc, D, params);
    params_view(&g, H, L, K, rc, D, grads);
    double loss_sum = 0.0;
    int st = 0;
    for (int gi = 0; gi < G && !st; ++gi) {
        double wl = 0.0;
        st = worker_body(&p, &g, gi, B, D, atom_ptr, pos, Z, dsidx, emask, fmask, energy, forces, denoise_flag, ntab,
                         rho, rho_has, mean, stdv, fstd, has, noise_sigma, noise_scheme, seed, step, lambda_e,
                         lambda_f, &wl);
        loss_sum += wl;
    }
    if (!st) {
        const double sG = 1.0 / (double)G; /* scale_params S/model.cpp:134-138 */
        for (int64_t k = 0; k < NP; ++k) grads[k] *= sG;
        const double loss = loss_sum / (double)G;
        double sq = 0.0; /* global_norm S/model.cpp:153-159 */
        for (int64_t k = 0; k < NP; ++k) sq += grads[k] * grads[k];
        const double gn = sqrt(sq);
        *out_loss = loss;
        *out_grad_norm = gn;
        if (out_grads) memcpy(out_grads, grads, sizeof(double) * NP);
        if (!isfinite(loss) || !isfinite(gn)) {
            set_err("non-finite loss or gradient");
            st = 5;
        } else {
            if (clip > 0.0 && gn > clip) {
                const double sc = clip / gn;
                for (int64_t k = 0; k < NP; ++k) grads[k] *= sc;
            }
            for (int64_t k = 0; k < NP; ++k) { /* RmsOptimizer::step S/trainer.cpp:37-53 */
                const double gk = grads[k];
                rms_v[k] = decay * rms_v[k] + (1.0 - decay) * gk * gk;
                params[k] -= lr * gk / (sqrt(rms_v[k]) + eps);
            }
        }
    }
    params_free(&p);
    params_free(&g);
    free(grads);
    return st;
}

/* ----------------------------------------------------------- scheduler --- */
static const int64_t* g_sort_key;
static int cmp_desc_then_index(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    const int64_t ax = g_sort_key[x], ay = g_sort_key[y];
    if (ax != ay) return ax > ay ? -1 : 1;
    return x < y ? -1 : (x > y);
}

/* greedy_assign S/scheduler.cpp:62-89: stable descending sort (== sort by
 * (atoms desc, position asc)), then LPT with a cap of B, ties to lowest worker. */
int lor_greedy_assign(const int64_t* atoms, int64_t n, int G, int B, int32_t* out) {
    if (G < 1 || B < 1) return set_err("greedy_assign: bad worker shape"), 1;
    if (n != (int64_t)G * B) return set_err("greedy_assign: need exactly workers*batch_per_worker samples"), 1;
    int64_t* order = malloc(sizeof(int64_t) * n);
    for (int64_t k = 0; k < n; ++k) order[k] = k;
    g_sort_key = atoms;
    qsort(order, (size_t)n, sizeof(int64_t), cmp_desc_then_index);
    int64_t* load = calloc((size_t)G, sizeof(int64_t));
    int* count = calloc((size_t)G, sizeof(int));
    for (int64_t q = 0; q < n; ++q) {
        const int64_t pos = order[q];
        int best = -1;
        for (int g = 0; g < G; ++g) {
            if (count[g] >= B) continue;
            if (best < 0 || load[g] < load[best]) best = g;
        }
        out[pos] = best;
        load[best] += atoms[pos];
        ++count[best];
    }
    free(order), free(load), free(count);
    return 0;
}

typedef struct {
    int64_t sample, atoms, split, chunk_rank;
} Sched;

/* pack_batch S/scheduler.cpp:43-58: worker-major, input order within a worker. */
static void pack_batch(const Sched* flat, const int32_t* assign, int64_t bs, int G, int64_t* o, int64_t* sample,
                       int32_t* worker, int64_t* oatoms, int64_t* split, int64_t* chunk_rank, int64_t* wa) {
    for (int g = 0; g < G; ++g) {
        wa[g] = 0;
        for (int64_t p = 0; p < bs; ++p) {
            if (assign[p] != g) continue;
            sample[*o] = flat[p].sample;
            worker[*o] = g;
            oatoms[*o] = flat[p].atoms;
            split[*o] = flat[p].split;
            chunk_rank[*o] = flat[p].chunk_rank;
            wa[g] += flat[p].atoms;
            ++*o;
        }
    }
}

int64_t lor_plan(const int64_t* atoms, int64_t n, int G, int B, int S, uint64_t seed, int mode, int64_t* sample,
                 int32_t* worker, int64_t* oatoms, int64_t* split, int64_t* chunk_rank, int64_t* worker_atoms,
                 int64_t* dropped) {
    if (G < 1) return set_err("schedule: workers must be >= 1"), -1;
    if (B < 1) return set_err("schedule: batch_per_worker must be >= 1"), -1;
    if (S < 1) return set_err("schedule: num_splits must be >= 1"), -1;
    for (int64_t k = 0; k < n; ++k)
        if (atoms[k] < 1) return set_err("schedule: atom counts must be >= 1"), -1;
    Rng r;
    rng_init(&r, seed);
    int64_t* perm = malloc(sizeof(int64_t) * (n ? n : 1));
    rng_permutation(&r, n, perm);
    const int64_t bs = (int64_t)G * B;
    Sched* flat = malloc(sizeof(Sched) * bs);
    int32_t* assign = malloc(sizeof(int32_t) * bs);
    int64_t* batoms = malloc(sizeof(int64_t) * bs);
    int64_t o = 0, nb = 0;
    *dropped = 0;
    if (mode == 0) { /* plan_balanced S/scheduler.cpp:91-158 */
        int64_t* sptr = malloc(sizeof(int64_t) * (S + 1));
        sptr[0] = 0;
        for (int64_t s = 0; s < S; ++s) sptr[s + 1] = sptr[s] + n / S + (s < n % S ? 1 : 0);
        g_sort_key = atoms;
        for (int64_t s = 0; s < S; ++s) /* sort by (atoms desc, id asc) */
            qsort(perm + sptr[s], (size_t)(sptr[s + 1] - sptr[s]), sizeof(int64_t), cmp_desc_then_index);
        int64_t max_ranks = 0;
        for (int64_t s = 0; s < S; ++s) {
            const int64_t len = sptr[s + 1] - sptr[s], ranks = len / G;
            *dropped += len - ranks * G;
            if (ranks > max_ranks) max_ranks = ranks;
        }
        Sched* stream = malloc(sizeof(Sched) * (n ? n : 1));
        int64_t ns = 0;
        for (int64_t rk = 0; rk < max_ranks; ++rk)
            for (int64_t s = 0; s < S; ++s) {
                const int64_t len = sptr[s + 1] - sptr[s];
                if ((rk + 1) * G > len) continue;
                for (int64_t k = rk * G; k < (rk + 1) * G; ++k) {
                    const int64_t id = perm[sptr[s] + k];
                    stream[ns++] = (Sched){id, atoms[id], s, rk};
                }
            }
        const int64_t full = ns / bs;
        *dropped += ns - full * bs;
        for (int64_t b = 0; b < full; ++b) {
            for (int64_t p = 0; p < bs; ++p) flat[p] = stream[b * bs + p], batoms[p] = flat[p].atoms;
            lor_greedy_assign(batoms, bs, G, B, assign);
            pack_batch(flat, assign, bs, G, &o, sample, worker, oatoms, split, chunk_rank, worker_atoms + nb * G);
            ++nb;
        }
        free(stream);
        free(sptr);
    } else { /* plan_naive S/scheduler.cpp:160-199 */
        const int64_t full = n / bs;
        *dropped = n - full * bs;
        for (int64_t b = 0; b < full; ++b) {
            for (int64_t p = 0; p < bs; ++p) {
                const int64_t id = perm[b * bs + p];
                flat[p] = (Sched){id, atoms[id], 0, (b * bs + p) / G};
                batoms[p] = flat[p].atoms;
            }
            if (mode == 1) lor_greedy_assign(batoms, bs, G, B, assign);
            else
                for (int64_t p = 0; p < bs; ++p) assign[p] = (int32_t)(p / B);
            pack_batch(flat, assign, bs, G, &o, sample, worker, oatoms, split, chunk_rank, worker_atoms + nb * G);
            ++nb;
        }
    }
    free(perm), free(flat), free(assign), free(batoms);
    return nb;
}

typedef struct {
    int64_t split, rank, atoms;
} ChunkKey;
static int cmp_chunk(const void* a, const void* b) {
    const ChunkKey *x = a, *y = b;
    if (x->split != y->split) return x->split < y->split ? -1 : 1;
    if (x->rank != y->rank) return x->rank < y->rank ? -1 : 1;
    return 0;
}

/* schedule_metrics S/scheduler.cpp:205-251 over the flat plan arrays. */
void lor_schedule_metrics(int64_t nbatches, int G, int B, const int32_t* worker, const int64_t* atoms,
                          const int64_t* split, const int64_t* chunk_rank, double* max_imb, double* mean_imb,
                          int64_t* mono, int64_t* growth) {
    const int64_t bs = (int64_t)G * B;
    double mx = 0.0, mean_sum = 0.0;
    int64_t* peak = calloc((size_t)G, sizeof(int64_t));
    int64_t* tot = calloc((size_t)G, sizeof(int64_t));
    int64_t grow = 0;
    for (int64_t st = 0; st < nbatches; ++st) {
        memset(tot, 0, sizeof(int64_t) * G);
        for (int64_t p = 0; p < bs; ++p) tot[worker[st * bs + p]] += atoms[st * bs + p];
        int64_t sum = 0, pk = 0;
        for (int g = 0; g < G; ++g) {
            sum += tot[g];
            if (tot[g] > pk) pk = tot[g];
            if (tot[g] > peak[g]) ++grow, peak[g] = tot[g];
        }
        const double mean = (double)sum / (double)G;
        const double imb = mean > 0.0 ? (double)pk / mean : 1.0;
        if (imb > mx) mx = imb;
        mean_sum += imb;
    }
    if (nbatches > 0) mean_sum /= (double)nbatches;
    else mx = mean_sum = 1.0;
    const int64_t total = nbatches * bs;
    ChunkKey* ck = malloc(sizeof(ChunkKey) * (total ? total : 1));
    for (int64_t k = 0; k < total; ++k) ck[k] = (ChunkKey){split[k], chunk_rank[k], atoms[k]};
    qsort(ck, (size_t)total, sizeof(ChunkKey), cmp_chunk);
    int64_t viol = 0, prev_split = -1, prev_total = 0;
    for (int64_t k = 0; k < total;) {
        int64_t e = k, t = 0;
        while (e < total && ck[e].split == ck[k].split && ck[e].rank == ck[k].rank) t += ck[e++].atoms;
        if (ck[k].split == prev_split && t > prev_total) ++viol;
        prev_split = ck[k].split;
        prev_total = t;
        k = e;
    }
    *max_imb = mx;
    *mean_imb = mean_sum;
    *mono = viol;
    *growth = grow;
    free(ck), free(peak), free(tot);
}

/* ------------------------------------------------------- trace/dataset --- */
static int64_t lognormal_draw(double mode, double sigma, Rng* r) { /* S/trace.cpp:40-45 */
    const double mu = log(mode) + sigma * sigma;
    return llround(exp(rng_normal_ms(r, mu, sigma)));
}

int lor_make_trace(int kind, int64_t count, int64_t min_atoms, int64_t max_atoms, double constant_atoms, double mode,
                   double sigma, double mode_a, double sigma_a, double mode_b, double sigma_b, double weight_a,
                   uint64_t seed, int64_t* out) { /* S/trace.cpp:50-76 */
    if (count < 1) return set_err("trace: count must be >= 1"), 1;
    if (min_atoms < 1 || max_atoms < min_atoms) return set_err("trace: bad atom bounds"), 1;
    if (!(constant_atoms >= 1.0) || !(mode >= 1.0) || !(mode_a >= 1.0) || !(mode_b >= 1.0))
        return set_err("trace: modes must be >= 1"), 1;
    if (!(sigma > 0.0) || !(sigma_a > 0.0) || !(sigma_b > 0.0)) return set_err("trace: sigmas must be positive"), 1;
    if (!(weight_a >= 0.0 && weight_a <= 1.0)) return set_err("trace: weight_a must be in [0, 1]"), 1;
    Rng r;
    rng_init(&r, seed);
    for (int64_t k = 0; k < count; ++k) {
        int64_t v = 0;
        switch (kind) {
            case 0: v = llround(constant_atoms); break;
            case 1: v = min_atoms + (int64_t)rng_bounded(&r, (uint64_t)(max_atoms - min_atoms + 1)); break;
            case 2: v = lognormal_draw(mode, sigma, &r); break;
            default:
                v = rng_uniform(&r) < weight_a ? lognormal_draw(mode_a, sigma_a, &r) : lognormal_draw(mode_b, sigma_b, &r);
                break;
        }
        out[k] = v < min_atoms ? min_atoms : (v > max_atoms ? max_atoms : v);
    }
    return 0;
}

int lor_temperature_counts(const double* sizes, int k, double T, double* out) { /* S/dataset.cpp:39-52 */
    if (k < 1) return set_err("temperature_counts: no subset sizes"), 1;
    if (!(T >= 1.0)) return set_err("temperature_counts: temperature must be >= 1"), 1;
    double nmax = 0.0;
    for (int q = 0; q < k; ++q) {
        if (!(sizes[q] > 0.0)) return set_err("temperature_counts: sizes must be positive"), 1;
        nmax = fmax(nmax, sizes[q]);
    }
    const double inv_t = 1.0 / T;
    for (int q = 0; q < k; ++q) out[q] = pow(nmax, 1.0 - inv_t) * pow(sizes[q], inv_t);
    return 0;
}

int64_t lor_build_epoch_index(const double* repeats, const int64_t* sizes, int k, uint64_t seed, int64_t cap,
                              int32_t* out_subset, int64_t* out_sample) { /* S/dataset.cpp:61-83 */
    int64_t total_all = 0;
    for (int q = 0; q < k; ++q) {
        if (sizes[q] <= 0) return set_err("build_epoch_index: subset sizes must be positive"), -1;
        const int64_t t = llround(repeats[q]);
        if (t < 0) return set_err("build_epoch_index: negative repeat count"), -1;
        total_all += t;
    }
    int32_t* es = malloc(sizeof(int32_t) * (total_all ? total_all : 1));
    int64_t* ex = malloc(sizeof(int64_t) * (total_all ? total_all : 1));
    int64_t e = 0;
    for (int q = 0; q < k; ++q) {
        const int64_t n = sizes[q], total = llround(repeats[q]);
        const int64_t base = total / n, extra = total % n;
        for (int64_t s = 0; s < n; ++s) {
            const int64_t copies = base + (s < extra ? 1 : 0);
            for (int64_t c = 0; c < copies; ++c) es[e] = q, ex[e] = s, ++e;
        }
    }
    Rng r;
    rng_init(&r, seed);
    for (int64_t m = e; m > 1; --m) {
        const int64_t j = (int64_t)rng_bounded(&r, (uint64_t)m);
        const int32_t ts = es[m - 1];
        es[m - 1] = es[j], es[j] = ts;
        const int64_t tx = ex[m - 1];
        ex[m - 1] = ex[j], ex[j] = tx;
    }
    for (int64_t q = 0; q < e && q < cap; ++q) out_subset[q] = es[q], out_sample[q] = ex[q];
    free(es), free(ex);
    return e;
}

/* Morse generator, S/dataset.cpp:121-230, default PairTable (fallback only). */
static const double kDepth = 1.0, kStiff = 2.2, kReq = 1.9;

static double vnorm3(double x, double y, double z) { return sqrt(x * x + y * y + z * z); }

static double morse_energy(int n, const double* x) {
    double e = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            const double r = vnorm3(x[3 * i] - x[3 * j], x[3 * i + 1] - x[3 * j + 1], x[3 * i + 2] - x[3 * j + 2]);
            const double g = 1.0 - exp(-kStiff * (r - kReq));
            e += kDepth * (g * g - 1.0);
        }
    return e;
}

static void morse_forces(int n, const double* x, double* f) {
    memset(f, 0, sizeof(double) * 3 * n);
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            const double d0 = x[3 * i] - x[3 * j], d1 = x[3 * i + 1] - x[3 * j + 1], d2 = x[3 * i + 2] - x[3 * j + 2];
            const double r = vnorm3(d0, d1, d2);
            const double e = exp(-kStiff * (r - kReq));
            const double dv = 2.0 * kDepth * (1.0 - e) * kStiff * e;
            const double s = -dv / r;
            const double f0 = s * d0, f1 = s * d1, f2 = s * d2;
            f[3 * i] = f[3 * i] + f0, f[3 * i + 1] = f[3 * i + 1] + f1, f[3 * i + 2] = f[3 * i + 2] + f2;
            f[3 * j] = f[3 * j] - f0, f[3 * j + 1] = f[3 * j + 1] - f1, f[3 * j + 2] = f[3 * j + 2] - f2;
        }
}

static int draw_atom_count(double mode, double sigma, int mn, int mx, Rng* r) { /* :150-157 */
    const double mu = log(mode) + sigma * sigma;
    const double v = exp(rng_normal_ms(r, mu, sigma));
    const int rounded = (int)llround(v);
    return rounded < mn ? mn : (rounded > mx ? mx : rounded);
}

int lor_synth_counts(int64_t count, double mode, double sigma, int min_atoms, int max_atoms, uint64_t seed,
                     int64_t* atom_ptr) {
    atom_ptr[0] = 0;
    for (int64_t s = 0; s < count; ++s) {
        Rng r;
        rng_init(&r, lor_mix_seed(seed, (uint64_t)s));
        atom_ptr[s + 1] = atom_ptr[s] + draw_atom_count(mode, sigma, min_atoms, max_atoms, &r);
    }
    return 0;
}

int lor_synth_fill(int task, int64_t count, double mode, double sigma, int min_atoms, int max_atoms,
                   const int32_t* elements, int nelem, int relax_steps, double relax_step, double energy_scale,
                   const int32_t* off_z, const double* off_v, int noff, uint64_t seed, const int64_t* atom_ptr,
                   double* pos, int32_t* Z, uint8_t* emask, uint8_t* fmask, double* energy, double* forces) {
    for (int64_t s = 0; s < count; ++s) { /* make_sample S/dataset.cpp:210-230 */
        Rng r;
        rng_init(&r, lor_mix_seed(seed, (uint64_t)s));
        const int n = draw_atom_count(mode, sigma, min_atoms, max_atoms, &r);
        double* x = pos + 3 * atom_ptr[s];
        int32_t* z = Z + atom_ptr[s];
        /* random_cluster :161-193 */
        const double min_sep = 0.8 * kReq;
        double radius = 0.75 * kReq * cbrt((double)n);
        for (int a = 0; a < n; ++a) {
            double p0 = 0, p1 = 0, p2 = 0;
            for (int attempt = 0;; ++attempt) {
                p0 = rng_uniform_in(&r, -radius, radius);
                p1 = rng_uniform_in(&r, -radius, radius);
                p2 = rng_uniform_in(&r, -radius, radius);
                if (vnorm3(p0, p1, p2) > radius) continue;
                int ok = 1;
                for (int q = 0; q < a; ++q)
                    if (vnorm3(p0 - x[3 * q], p1 - x[3 * q + 1], p2 - x[3 * q + 2]) < min_sep) {
                        ok = 0;
                        break;
                    }
                if (ok) break;
                if (attempt >= 200) {
                    radius *= 1.1;
                    attempt = 0;
                }
            }
            x[3 * a] = p0, x[3 * a + 1] = p1, x[3 * a + 2] = p2;
            z[a] = elements[rng_bounded(&r, (uint64_t)nelem)];
        }
        /* relax :195-208 */
        double* f = forces + 3 * atom_ptr[s];
        for (int step = 0; step < relax_steps; ++step) {
            morse_forces(n, x, f);
            for (int a = 0; a < n; ++a) {
                double m0 = relax_step * f[3 * a], m1 = relax_step * f[3 * a + 1], m2 = relax_step * f[3 * a + 2];
                const double m = vnorm3(m0, m1, m2);
                if (m > 0.25) {
                    const double sc = 0.25 / m;
                    m0 = sc * m0, m1 = sc * m1, m2 = sc * m2;
                }
                x[3 * a] = x[3 * a] + m0, x[3 * a + 1] = x[3 * a + 1] + m1, x[3 * a + 2] = x[3 * a + 2] + m2;
            }
        }
        emask[s] = 0, fmask[s] = 0, energy[s] = 0.0;
        memset(f, 0, sizeof(double) * 3 * n);
        if (task == 2) continue; /* denoising: structures only */
        double e = energy_scale * morse_energy(n, x);
        for (int a = 0; a < n; ++a)
            for (int q = 0; q < noff; ++q)
                if (off_z[q] == z[a]) {
                    e += off_v[q];
                    break;
                }
        energy[s] = e;
        emask[s] = 1;
        if (task == 0) {
            morse_forces(n, x, f);
            for (int k = 0; k < 3 * n; ++k) f[k] = energy_scale * f[k];
            fmask[s] = 1;
        }
    }
    return 0;
}

/* Worker g's contribution alone (its loss and gradient SUM before the /G), for
 * checking a data-parallel decomposition: sum over g of these == the step body. */
int lor_worker_step(int H, int L, int K, double rc, int D, int G, int B, int g, const int64_t* atom_ptr,
                    const double* pos, const int32_t* Z, const int32_t* dsidx, const uint8_t* emask,
                    const uint8_t* fmask, const double* energy, const double* forces, const uint8_t* denoise_flag,
                    int ntab, const double* rho, const uint8_t* rho_has, const double* mean, const double* stdv,
                    const double* fstd, const uint8_t* has, double noise_sigma, int noise_scheme, uint64_t seed,
                    int64_t step, double lambda_e, double lambda_f, const double* params, double* out_loss,
                    double* out_grads) {
    if (validate_config(H, L, K, rc, D)) return 1;
    if (g < 0 || g >= G) return set_err("worker_step: bad worker"), 1;
    const int64_t NP = lor_param_count(H, L, K, D);
    memset(out_grads, 0, sizeof(double) * NP);
    Params p, gg;
    params_view(&p, H, L, K, rc, D, (double*)params);
    params_view(&gg, H, L, K, rc, D, out_grads);
    const int st = worker_body(&p, &gg, g, B, D, atom_ptr, pos, Z, dsidx, emask, fmask, energy, forces, denoise_flag,
                               ntab, rho, rho_has, mean, stdv, fstd, has, noise_sigma, noise_scheme, seed, step,
                               lambda_e, lambda_f, out_loss);
    params_free(&p);
    params_free(&gg);
    return st;
}
