// device.cuh - device-side state of one lamm_ctx and the helpers shared by the
// sm_100a kernels (kernels.cuh) and the host orchestration (device.cu).
//
// HBM layout of one device-batch (all row-major, atoms in batch order, every
// sample's atoms contiguous — the CSR the host packs):
//   positions  x/y/z        fp64 SoA [N]           (bit-exact neighbour test)
//   edges      row_ptr      int32 [N+1]            (CSR by destination atom i,
//              col          int32 [P]               j ascending = reference order)
//              geo          float4 [P]  {u_x,u_y,u_z,fcut}
//              dst          int32 [P]               (destination i of each edge)
//              rbf          fp32 [P][K]             (fcut * Gaussians of the fp64 distance)
//   features   t[l], h[l]   fp32 [N][H]  l = 1..L   (t = tanh h; t[0] = tanh(E[Z]))
//              mu[l]        fp32 [N][H]  l = 0..L-1 (tanh of the message)
//   heads      e_atom       fp32 [N][NS][D]        (per-atom energy, one partial per node-GEMM
//                                                   column split)
//              F            fp32 [N][D][3]
//   backward   gh, gm       fp32 [N][H]
//              Q            fp32 [N][H+K+1]         (per-atom force-head terms)
//   gradients  partials     fp32 [ncta][tensor]     (deterministic per-CTA sums)
//              grads        fp32 [NP + 4]           (flat for_each_tensor order +
//                                                    loss hi/lo, overflow, count)
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace lamm_b200 {

constexpr int kMaxLayers = 8;
constexpr int kMaxHeads = 16;
constexpr int kMaxZ = 118;

// Per-step scalars that live in device memory so one captured CUDA graph can
// be replayed for device-batches of any size.
// Samples with more atoms than this get a cell list (k_prep bins, k_cell_count
// counts, k_nbr_fill walks the 27 neighbour cells); smaller ones are swept
// brute force by the sample's own block.
constexpr int kSmallAtoms = 128;
// Cell-list samples up to this size keep each row's hit bitmask (kMaskAtoms / 32
// words) between k_cell_count and k_nbr_fill.
constexpr int kMaskAtoms = 2048;
constexpr int kMaskWords = kMaskAtoms / 32;

// Uniform grid over one sample: non-periodic — the bounding box cut into cells of
// width >= rc (1 + 1e-9); periodic — n[k] slabs of fractional coordinate k, each
// at least rc (1 + 1e-9) wide perpendicular to the face. Either way two atoms
// within rc sit in the same or adjacent cells (wrapped when periodic), so the
// exact pair test over the neighbour cells finds the brute-force pair set.
struct CellGrid {
    double lo[3], scale[3];  // non-periodic: cell k = floor((x_k - lo_k) * scale_k)
    int n[3], periodic;
    int base, pad;           // region of the sample's cell offsets in Dev::cstart
};

struct StepHeader {
    int32_t B, N, P, overflow;   // P written by k_prep; overflow if P > capacity
    int32_t me, mf;              // this rank's sum m_E, sum m_F (after denoise relabelling)
    int32_t nslots, status;      // distinct atomic numbers; non-finite flag
    int32_t workers, n_large;    // n_large: samples k_cell_count counts (above kSmallAtoms or periodic)
    int32_t chain, pad2;         // chain: submitted by lamm_train_step_submit (in-flight poison applies)
    double lambda_e, lambda_f;
    double loss_energy, loss_force, loss_total;  // this rank's Eq. (5) breakdown
    double grad_norm, clip_scale, global_loss;
    uint32_t done_counter, large_done;
    // byte offsets of the staged input arrays inside the upload blob (the blob
    // starts with this header), see device.cu:pack_batch
    int64_t off_atom_ptr, off_pos, off_Z, off_z2s, off_dsidx, off_emask, off_fmask, off_denoise, off_E, off_F,
        off_noise, off_cell, blob_bytes;  // off_cell: [B] x {periodic flag, cell[9], cell^-1[9]} (0: none)
};

struct Dev {
    int H, L, K, D;
    double rc;
    int64_t Ncap, Bcap, Pcap;
    StepHeader* hdr;
    // batch (uploaded blob + prep outputs)
    const int64_t* atom_ptr;
    const double* pos_in;      // [3N] AoS from the host
    const int32_t* Z;          // [N]
    const int32_t* zslot;      // [N]  slot of Z among the batch's distinct Z
    const int32_t* z_to_slot;  // [119] (-1: absent)
    const int32_t* dsidx;      // [B]
    const uint8_t* emask;      // [B]  effective m_E (0 for denoising samples)
    const uint8_t* fmask;      // [B]  effective m_F (1 for denoising samples)
    const uint8_t* denoise;    // [B]
    const double* E_raw;       // [B]
    const double* F_raw;       // [3N]
    const double* noise;       // [3N] raw Gaussian displacement draws (denoising samples)
    int32_t* sample_of;        // [N]
    int32_t* chan;             // [N]  head (dataset index) of the atom's sample
    double *x, *y, *z;         // [N] fp64 (noisy) positions, SoA
    double* En;                // [B]  normalized energy labels
    double* Fn;                // [3N] normalized force labels
    int use_table, denoise_scheme, ntab;
    const double* rho;         // [ntab][119]
    const uint8_t* rho_has;
    const double *tmean, *tstd, *tfstd;
    const uint8_t* thas;
    // edges
    int32_t *cnt, *row_ptr, *col, *dst;
    int32_t* colz;             // [P] Z_j - 1 of each edge's source (layer-0 message rows)
    int32_t *lptr, *stot, *soff;  // per-atom row offset inside its sample, per-sample edge totals / offsets
    uint32_t* segw;            // bit p set: edge p is the first of its destination atom
    int32_t* part_lo;          // [Q+1] atom partitions of the edge kernels, balanced on edges + kAtomCost per atom
    // cell lists of the large samples (k_prep bins, k_cell_count / k_nbr_fill walk)
    CellGrid* cgrid;           // [B]
    int32_t* acell;            // [N]  linear cell of the atom inside its sample's grid
    int32_t* cstart;           // [4 N + 65 B + 1] per-sample cell offsets (region 4 lo + 65 s)
    double4* cpos;             // [N]  the sample's atoms ordered by cell: x, y, z, j (bits)
    uint32_t* sdone;           // [B]  atoms of the sample counted (k_cell_count)
    uint32_t* cmask;           // [N][kMaskWords] hit bitmask of a row of a sample <= kMaskAtoms
    float4* geo;
    float2* sij;               // [P] train step: fcut (gF_i - gF_j).u_ij and gF_i.u_ij (k_loss, for k_edge_head)
    float* rbf;                // [P][K] fcut * Gaussians, canonical tcgen05 layout, tf32 hi part
    float* rbfl;               //        ... and the fp32 lo remainder
    float* rbfp;               // [P][K] fcut * Gaussians, edge-major (FFMA consumers)
    double *dist64, *unit64;
    int export64;
    // fp32 working parameters
    const float* emb;        // [118][H]
    const float* tanh_emb;   // [118][H]
    const float* wf[kMaxLayers];  // [H][K]
    const float* wu[kMaxLayers];  // [H][H]  (row b = output, col a = input)
    const float* we;         // [H][D]
    const float* wfh;        // [2H+K][D]
    // activations
    float* t[kMaxLayers + 1];
    float* h[kMaxLayers + 1];
    float* mu[kMaxLayers];
    float* F;
    float* Yf;               // [N][3H + 3 + 3K] per-atom force-head features (k_edge_force)
    double* Epred;           // [B][D]
    // loss gradients
    float* gE;               // [B][D]
    float* gF;               // [N][D][3]
    float4* gFc;             // [N] dL/dF of the atom's own head (loss path), w = 0
    double* eatom;           // [N] sum_a h^L[i,a] W_e[a,d_i] (train step: own head)
    double* fterm;           // [N] the atom's Eq. (5) force term m_F w_F / n ||dF||
    double* fw;              // [N] m_F lambda_F / (sum m_F * n) of the atom's sample (k_prep)
    double* sample_terms;    // [B][2]
    double* block_scratch;   // reduction scratch
    // backward
    float *gh, *gm, *Q;
    float* part_wf[kMaxLayers];
    float* part_wu[kMaxLayers];
    float* part_head;
    float* part_emb;
    int ncta_edge, ncta_gemm, ncta_red;
    float* grads;            // [NP + 4]
    // fp64 master state
    double *p64, *v64;
    const double* g64_in;    // optional fp64 gradient input for the optimizer
    int g64_loss;            // g64_in carries the loss terms at [NP], [NP + 1] (simulated workers)
    double* g64_acc;         // fp64 worker-gradient accumulator [NP + 4]
    float* p32;              // [NP] fp32 working copy (emb/wf/wu/... point into it)
    float* tanh_emb_w;       // writable alias of tanh_emb
    int64_t NP;
    int32_t emb_rows;
    unsigned int* anomaly;   // [0] steps whose update was skipped, [8] in-flight poison, [16..] grid barrier
    float* wpack;            // [L][4][H*H] packed tcgen05 weight operands (k_pack_weights)
};

// Programmatic dependent launch: every kernel of the step is launched with
// programmatic stream serialization, so its CTAs may start while the previous
// kernel drains. pdl_enter() waits until that kernel has completed (its writes
// visible) and immediately lets the next kernel launch. Code before pdl_enter()
// may only read data produced two or more kernels back (weights, the CSR
// partition) and must not write anything a running kernel could read.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Periodic cells: per sample 24 doubles {flag, cell[9] (rows = lattice vectors),
// cell^-1[9], m[3], nimg, 0} in the staged blob. flag 1: every periodic width is
// at least 2 rc (m = 0): the minimum image, cell lists above kSmallAtoms; flag 2:
// several images per pair (m_k >= 1) or an open axis (m_k = -1): brute force over
// (j, image). The image n of a pair uses
//   f_k = sum_c d_c cinv[c][k];  f_k -= rint(f_k) (periodic axes);  f_k -= n_k;
//   d_c = sum_k f_k cell[k][c]
// left to right, correctly rounded (oracle/lamm_oracle.c:image_disp is the same;
// n = 0 gives min_image below bit for bit).
constexpr int kCellDoubles = 24;
constexpr int kMaxImages = 4096;

__host__ __device__ inline bool cell_inverse(const double* m, double* inv) {
    const double c00 = m[4] * m[8] - m[5] * m[7], c01 = m[5] * m[6] - m[3] * m[8], c02 = m[3] * m[7] - m[4] * m[6];
    const double c10 = m[2] * m[7] - m[1] * m[8], c11 = m[0] * m[8] - m[2] * m[6], c12 = m[1] * m[6] - m[0] * m[7];
    const double c20 = m[1] * m[5] - m[2] * m[4], c21 = m[2] * m[3] - m[0] * m[5], c22 = m[0] * m[4] - m[1] * m[3];
    const double det = (m[0] * c00 + m[1] * c01) + m[2] * c02;
    if (!(det != 0.0)) return false;
    const double cof[9] = {c00, c10, c20, c01, c11, c21, c02, c12, c22};  // adjugate, row-major
    for (int k = 0; k < 9; ++k) inv[k] = cof[k] / det;
    return true;
}

__device__ __forceinline__ void min_image(const double* cell, const double* ci, double& d0, double& d1, double& d2) {
    double f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double a = __dmul_rn(d0, ci[k]), b = __dmul_rn(d1, ci[3 + k]), c = __dmul_rn(d2, ci[6 + k]);
        f[k] = __dadd_rn(__dadd_rn(a, b), c);
        f[k] = __dsub_rn(f[k], rint(f[k]));
    }
    double o[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double a = __dmul_rn(f[0], cell[c]), b = __dmul_rn(f[1], cell[3 + c]), e = __dmul_rn(f[2], cell[6 + c]);
        o[c] = __dadd_rn(__dadd_rn(a, b), e);
    }
    d0 = o[0], d1 = o[1], d2 = o[2];
}

// Images of a flag-2 sample (cell + 18 holds m[3]) in two parts: the pair's
// fractional minimum-image displacement (once per (i, j)), then image n of it
// with the rounded squared distance (once per image).
__device__ __forceinline__ void image_frac(const double* cell, double d0, double d1, double d2, double (&f)[3]) {
    const double* ci = cell + 9;
    const double* m = cell + 18;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double a = __dmul_rn(d0, ci[k]), b = __dmul_rn(d1, ci[3 + k]), c = __dmul_rn(d2, ci[6 + k]);
        f[k] = __dadd_rn(__dadd_rn(a, b), c);
        if (m[k] >= 0.0) f[k] = __dsub_rn(f[k], rint(f[k]));
    }
}
__device__ __forceinline__ double image_sq(const double* cell, const double (&f)[3], int n0, int n1, int n2,
                                           double& d0, double& d1, double& d2) {
    const double g0 = __dsub_rn(f[0], static_cast<double>(n0)), g1 = __dsub_rn(f[1], static_cast<double>(n1)),
                 g2 = __dsub_rn(f[2], static_cast<double>(n2));
    double o[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double a = __dmul_rn(g0, cell[c]), b = __dmul_rn(g1, cell[3 + c]), e = __dmul_rn(g2, cell[6 + c]);
        o[c] = __dadd_rn(__dadd_rn(a, b), e);
    }
    d0 = o[0], d1 = o[1], d2 = o[2];
    return __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int N>
struct VecF {
    float v[N];
};

template <int N>
__device__ __forceinline__ VecF<N> ldv(const float* __restrict__ p) {
    VecF<N> r;
    if constexpr (N == 4) {
        const float4 q = *reinterpret_cast<const float4*>(p);
        r.v[0] = q.x, r.v[1] = q.y, r.v[2] = q.z, r.v[3] = q.w;
    } else if constexpr (N == 2) {
        const float2 q = *reinterpret_cast<const float2*>(p);
        r.v[0] = q.x, r.v[1] = q.y;
    } else {
#pragma unroll
        for (int c = 0; c < N; ++c) r.v[c] = p[c];
    }
    return r;
}

template <int N>
__device__ __forceinline__ void stv(float* p, const VecF<N>& r) {
    if constexpr (N == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
    } else if constexpr (N == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(r.v[0], r.v[1]);
    } else {
#pragma unroll
        for (int c = 0; c < N; ++c) p[c] = r.v[c];
    }
}

}  // namespace lamm_b200
