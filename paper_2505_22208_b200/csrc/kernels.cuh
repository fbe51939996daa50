// kernels.cuh - sm_100a kernels of the LaMM energy/force train step.
//
// One kernel per dependency level of the step (a level boundary is a grid-wide
// dependency: the next level gathers rows that any CTA may have produced).
// Every kernel is persistent-grid / grid-stride and reads the batch sizes from
// StepHeader in device memory, so the whole step is captured once as a CUDA
// graph and replayed for device-batches of any size.
//
// Reference semantics (S = /root/reference/proj/core/src):
//   k_prep .......... S/denoise.cpp:7-29 (centering) + S/loss.cpp:113-126 (normalize)
//                     + the per-atom pair counts of S/core.cpp:30-48
//   k_nbr_fill ...... S/core.cpp:30-48  (bit-exact fp64 pair test, i-major, j ascending)
//   k_energy/k_loss . S/model.cpp:208-218 + S/loss.cpp:140-213 (Eq. 5, per-rank mask denominators)
//   k_emb_grad ...... S/model.cpp:421-424
//   k_grad_reduce ... sum of the per-CTA gradient partials
//   (edge kernels in edge_kernels.cuh; tensor-core GEMMs and k_opt — S/trainer.cpp:319-327
//    + RmsOptimizer :37-53 — in gemm_kernels.cuh)
//
// Determinism: no floating-point atomics. Parameter gradients are reduced into
// per-CTA partials in a fixed order and summed across CTAs in index order by
// k_grad_reduce; the grid sizes are fixed per device, so a step is bit-for-bit
// reproducible run to run.
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"
#include "edge_kernels.cuh"
#include "umma.cuh"

namespace lamm_b200 {

constexpr double kPiD = 3.14159265358979323846;

// All kernels share one dynamic shared-memory symbol (extern __shared__ arrays
// of different element types would otherwise collide).
template <class T>
__device__ __forceinline__ T* dyn_smem() {
    extern __shared__ __align__(16) unsigned char lamm_smem_raw[];
    return reinterpret_cast<T*>(lamm_smem_raw);
}

// ----------------------------------------------------------------- prep ---
// One block per sample (grid-stride): denoise centering with the reference's
// sequential fp64 mean, noisy positions x + dx_eff, labels -dx_eff, label
// normalization, and the fixed-capacity copies of the staged batch arrays.
struct BatchArrays {
    int64_t* atom_ptr;
    int32_t *Z, *zslot, *z_to_slot, *dsidx;
    uint8_t *emask, *fmask, *denoise;
};

// ------------------------------------------------------- neighbour list ---
// Bit-exact with S/core.cpp:40-43: d = p_i - p_j, r = sqrt((dx*dx + dy*dy) + dz*dz)
// with every operation individually rounded (no FMA contraction), r < cutoff.
// cell: nullptr, or {cell[9], cell^-1[9]} of a periodic sample (minimum image)
__device__ __forceinline__ double pair_dist(double xi, double yi, double zi, double xj, double yj, double zj,
                                            double& dx, double& dy, double& dz, const double* cell = nullptr) {
    dx = __dsub_rn(xi, xj);
    dy = __dsub_rn(yi, yj);
    dz = __dsub_rn(zi, zj);
    if (cell) min_image(cell, cell + 9, dx, dy, dz);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

// The sample's periodic cell in the staged blob, or nullptr.
__device__ __forceinline__ const double* sample_cell(const Dev& d, int s) {
    const StepHeader& hd = *d.hdr;
    if (hd.off_cell == 0) return nullptr;
    const double* c = reinterpret_cast<const double*>(reinterpret_cast<const char*>(d.hdr) + hd.off_cell) +
                      static_cast<int64_t>(kCellDoubles) * s;
    return c[0] != 0.0 ? c + 1 : nullptr;
}


// Exclusive scan of one value per thread over a 128-thread block; *total gets
// the block sum. Uses 4 ints of shared scratch; ends with a barrier.
__device__ __forceinline__ int block_excl_scan128(int v, int* scratch, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) scratch[w] = incl;
    __syncthreads();
    int off = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) off += k < w ? scratch[k] : 0;
    *total = scratch[0] + scratch[1] + scratch[2] + scratch[3];
    __syncthreads();
    return off + incl - v;
}

// Also the CSR row offsets (S/core.cpp:30-48 order: i-major): each sample's
// block scans its atoms' pair counts (lptr = offset inside the sample, stot =
// sample total); the last block to finish scans the sample totals (soff), sets
// P / the capacity-overflow flag / row_ptr[N] / the CSR padding, so the
// neighbour fill can place every atom's row without a separate scan kernel.
// Q: edge-kernel partitions (k_nbr_fill cuts them while writing row_ptr).
__global__ void __launch_bounds__(128) k_prep(Dev d, BatchArrays out, int Q) {
    pdl_enter();
    const StepHeader& hd = *d.hdr;
    const char* base = reinterpret_cast<const char*>(d.hdr);
    const int B = hd.B;
    const int64_t* ap = reinterpret_cast<const int64_t*>(base + hd.off_atom_ptr);
    const double* pos = reinterpret_cast<const double*>(base + hd.off_pos);
    const int32_t* Z = reinterpret_cast<const int32_t*>(base + hd.off_Z);
    const int32_t* z2s = reinterpret_cast<const int32_t*>(base + hd.off_z2s);
    const int32_t* ds = reinterpret_cast<const int32_t*>(base + hd.off_dsidx);
    const uint8_t* em = reinterpret_cast<const uint8_t*>(base + hd.off_emask);
    const uint8_t* fm = reinterpret_cast<const uint8_t*>(base + hd.off_fmask);
    const uint8_t* dn = reinterpret_cast<const uint8_t*>(base + hd.off_denoise);
    const double* E = reinterpret_cast<const double*>(base + hd.off_E);
    const double* F = reinterpret_cast<const double*>(base + hd.off_F);
    const double* noise = reinterpret_cast<const double*>(base + hd.off_noise);
    if (blockIdx.x == 0) {
        for (int k = threadIdx.x; k < 119; k += blockDim.x) out.z_to_slot[k] = z2s[k];
        if (threadIdx.x == 0) out.atom_ptr[B] = ap[B];
    }
    {  // segment-start bits are OR-ed in by k_nbr_fill: clear the whole capacity
        const int64_t words = (((static_cast<int64_t>(d.Pcap) + kChunk + 16 + 7) / 8) * 8) / 32 + 32;
        for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < words;
             x += static_cast<int64_t>(gridDim.x) * blockDim.x)
            d.segw[x] = 0u;
    }
    __shared__ double mean[3];
    __shared__ int scan_scratch[4];
    __shared__ bool last;
    for (int s = blockIdx.x; s < B; s += gridDim.x) {
        const int64_t lo = ap[s], hi = ap[s + 1];
        const int dsi = ds[s];
        const bool is_dn = dn[s] != 0;
        if (threadIdx.x == 0) {
            out.atom_ptr[s] = lo;
            out.dsidx[s] = dsi;
            out.emask[s] = em[s];
            out.fmask[s] = fm[s];
            out.denoise[s] = dn[s];
            double m0 = 0.0, m1 = 0.0, m2 = 0.0;
            if (is_dn && d.denoise_scheme) {  // S/denoise.cpp:14-19, sequential sum then (1/n)*sum
                for (int64_t a = lo; a < hi; ++a) {
                    m0 = __dadd_rn(m0, noise[3 * a]);
                    m1 = __dadd_rn(m1, noise[3 * a + 1]);
                    m2 = __dadd_rn(m2, noise[3 * a + 2]);
                }
                const double sc = __ddiv_rn(1.0, static_cast<double>(hi - lo));
                m0 = __dmul_rn(sc, m0), m1 = __dmul_rn(sc, m1), m2 = __dmul_rn(sc, m2);
            }
            mean[0] = m0, mean[1] = m1, mean[2] = m2;
            double e = E[s];
            if (d.use_table && em[s]) {  // S/loss.cpp:117-121
                double total = 0.0;
                for (int64_t a = lo; a < hi; ++a)
                    if (d.rho_has[dsi * 119 + Z[a]]) total = __dadd_rn(total, d.rho[dsi * 119 + Z[a]]);
                e = __ddiv_rn(__dsub_rn(__dsub_rn(e, total), d.tmean[dsi]), d.tstd[dsi]);
            }
            d.En[s] = e;
        }
        __syncthreads();
        const double fs = d.use_table ? __ddiv_rn(1.0, d.tfstd[dsi]) : 1.0;
        for (int64_t a = lo + threadIdx.x; a < hi; a += blockDim.x) {
            d.sample_of[a] = s;
            d.chan[a] = dsi;
            out.Z[a] = Z[a];
            out.zslot[a] = z2s[Z[a]];
            double xyz[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double lab;
                if (is_dn) {
                    const double eff = d.denoise_scheme ? __dsub_rn(noise[3 * a + c], mean[c]) : noise[3 * a + c];
                    xyz[c] = __dadd_rn(pos[3 * a + c], eff);
                    lab = __dmul_rn(-1.0, eff);
                } else {
                    xyz[c] = pos[3 * a + c];
                    lab = F[3 * a + c];
                }
                d.Fn[3 * a + c] = d.use_table ? __dmul_rn(fs, lab) : lab;
            }
            d.x[a] = xyz[0], d.y[a] = xyz[1], d.z[a] = xyz[2];
        }
        __syncthreads();
        // neighbour counts of the sample (S/core.cpp:30-48), warp per atom, from the
        // positions this block just wrote (plain loads: visible after the barrier)
        const int lane = threadIdx.x & 31;
        const double* cell = sample_cell(d, s);
        for (int64_t i = lo + (threadIdx.x >> 5); i < hi; i += blockDim.x >> 5) {
            const double xi = d.x[i], yi = d.y[i], zi = d.z[i];
            int cnt = 0;
            for (int64_t j0 = lo; j0 < hi; j0 += 32) {
                const int64_t j = j0 + lane;
                bool in = false;
                if (j < hi && j != i) {
                    double dx, dy, dz;
                    in = pair_dist(xi, yi, zi, d.x[j], d.y[j], d.z[j], dx, dy, dz, cell) < d.rc;
                }
                cnt += __popc(__ballot_sync(0xffffffffu, in));
            }
            if (lane == 0) d.cnt[i] = cnt;
        }
        __syncthreads();
        int run = 0;  // the sample's row offsets, atoms in index order
        for (int64_t c0 = lo; c0 < hi; c0 += blockDim.x) {
            const int64_t a = c0 + threadIdx.x;
            const int v = a < hi ? d.cnt[a] : 0;
            int tot;
            const int ex = block_excl_scan128(v, scan_scratch, &tot);
            if (a < hi) d.lptr[a] = run + ex;
            run += tot;
        }
        if (threadIdx.x == 0) d.stot[s] = run;
    }
    // the last block: offsets of the samples, P, overflow, row_ptr[N], padding
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&d.hdr->done_counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    int run = 0;
    for (int c0 = 0; c0 < B; c0 += blockDim.x) {
        const int s = c0 + threadIdx.x;
        const int v = s < B ? d.stot[s] : 0;
        int tot;
        const int ex = block_excl_scan128(v, scan_scratch, &tot);
        if (s < B) d.soff[s] = run + ex;
        run += tot;
    }
    const int N = hd.N;
    const bool over = static_cast<int64_t>(run) > d.Pcap;
    if (threadIdx.x == 0) {
        d.hdr->P = run;
        d.hdr->overflow = over ? 1 : 0;
        d.row_ptr[N] = run;
        d.hdr->done_counter = 0;
    }
    // partitions: cut by k_nbr_fill when there are edges; all empty on overflow
    // (the step is discarded and rerun with more capacity); no edges: the last
    // partition walks every atom (edge-less begin/end)
    if (over || run == 0)
        for (int q = threadIdx.x; q < Q; q += blockDim.x) d.part_lo[q] = 0;
    if (threadIdx.x == 0) d.part_lo[Q] = over ? 0 : N;
    if (!over)  // CSR padding read by the edge kernels' block staging: valid source atom 0
        for (int x = threadIdx.x; x < kChunk + 8; x += blockDim.x) d.col[run + x] = 0, d.dst[run + x] = N;
}

// Same sweep as the count in k_prep; lanes that hold a neighbour compact into the CSR
// row with popc(ballot & lanes_below). Edge geometry is computed in fp64 and
// rounded once: unit (1/r)*d (S/core.cpp:43), fcut (S/model.cpp:17), Gaussians
// (S/model.cpp:20-27).
template <int K>
__global__ void __launch_bounds__(256) k_nbr_fill(Dev d, int Q) {
    pdl_enter();
    if (d.hdr->overflow) return;
    const int N = d.hdr->N;
    const int64_t P = d.hdr->P;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const double width = d.rc / static_cast<double>(K - 1);
    const float wf = static_cast<float>(width), invf = static_cast<float>(1.0 / (2.0 * width * width));
    const float rc_inv = static_cast<float>(1.0 / d.rc);
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
        const int s = d.sample_of[i];
        const int lo = static_cast<int>(d.atom_ptr[s]), hi = static_cast<int>(d.atom_ptr[s + 1]);
        const double xi = d.x[i], yi = d.y[i], zi = d.z[i];
        const double* cell = sample_cell(d, s);
        int base = d.soff[s] + d.lptr[i];
        if (lane == 0) {
            const int ci = d.cnt[i];
            d.row_ptr[i] = base;
            if (ci > 0) atomicOr(d.segw + (base >> 5), 1u << (base & 31));
            // edge-kernel partitions: part_lo[q] = first atom with row_ptr >= floor(P q / Q)
            if (P > 0) {
                const int64_t prev = i == 0 ? -1 : base - d.cnt[i - 1];  // row_ptr[i - 1]
                const int64_t qlo = i == 0 ? 0 : ((prev + 1) * Q + P - 1) / P;
                int64_t qhi = ((static_cast<int64_t>(base) + 1) * Q + P - 1) / P - 1;
                if (qhi > Q - 1) qhi = Q - 1;
                for (int64_t q = qlo; q <= qhi; ++q) d.part_lo[q] = i;
                if (i == N - 1)  // targets in (row_ptr[N-1], P] start at atom N
                    for (int64_t q = ((static_cast<int64_t>(base) + 1) * Q + P - 1) / P; q < Q; ++q) d.part_lo[q] = N;
            }
        }
        for (int j0 = lo; j0 < hi; j0 += 32) {
            const int j = j0 + lane;
            bool in = false;
            double dx = 0, dy = 0, dz = 0, r = 0;
            if (j < hi && j != i) {
                r = pair_dist(xi, yi, zi, d.x[j], d.y[j], d.z[j], dx, dy, dz, cell);
                in = r < d.rc;
            }
            const unsigned mask = __ballot_sync(0xffffffffu, in);
            if (in) {
                const int p = base + __popc(mask & ((1u << lane) - 1u));
                d.col[p] = j;
                d.dst[p] = i;
                const double sc = __ddiv_rn(1.0, r);
                const double ux = __dmul_rn(sc, dx), uy = __dmul_rn(sc, dy), uz = __dmul_rn(sc, dz);
                // fcut and the Gaussians feed the fp32 model: evaluated in fp32 from the
                // once-rounded distance (relative error ~1e-6, far inside the 1e-4 bar)
                const float rf = static_cast<float>(r);
                const float fc = 0.5f * (cospif(rf * rc_inv) + 1.f);
                d.geo[p] = make_float4(static_cast<float>(ux), static_cast<float>(uy), static_cast<float>(uz), fc);
                float rb[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float dd = rf - wf * static_cast<float>(k);
                    rb[k] = fc * expf(-dd * dd * invf);  // fcut folded in
                }
#pragma unroll
                for (int q = 0; q < K / 4; ++q) {  // canonical tcgen05 layout, tf32 hi + fp32 lo
                    float4 hi, lo;
                    umma::split_tf32(rb[4 * q], hi.x, lo.x);
                    umma::split_tf32(rb[4 * q + 1], hi.y, lo.y);
                    umma::split_tf32(rb[4 * q + 2], hi.z, lo.z);
                    umma::split_tf32(rb[4 * q + 3], hi.w, lo.w);
                    const int64_t o = rbf_idx<K>(p, 4 * q);
                    *reinterpret_cast<float4*>(d.rbf + o) = hi;
                    *reinterpret_cast<float4*>(d.rbfl + o) = lo;
                    *reinterpret_cast<float4*>(d.rbfp + static_cast<int64_t>(p) * K + 4 * q) =
                        make_float4(rb[4 * q], rb[4 * q + 1], rb[4 * q + 2], rb[4 * q + 3]);
                }
                if (d.export64) {
                    d.dist64[p] = r;
                    d.unit64[3 * static_cast<int64_t>(p)] = ux;
                    d.unit64[3 * static_cast<int64_t>(p) + 1] = uy;
                    d.unit64[3 * static_cast<int64_t>(p) + 2] = uz;
                }
            }
            base += __popc(mask);
        }
    }
}

template <int K>
__device__ __forceinline__ void load_rbf(const float* __restrict__ src, float (&rb)[K]) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int k = 0; k < K / 4; ++k) {
        const float4 q = __ldg(s4 + k);
        rb[4 * k] = q.x, rb[4 * k + 1] = q.y, rb[4 * k + 2] = q.z, rb[4 * k + 3] = q.w;
    }
}

// ---------------------------------------------------------------- energy ---
// Per-sample energies for every head (S/model.cpp:208-218),
// E_s^d = sum_{i in s} sum_a W_e[a,d] h^L_ia: thread a accumulates its channel
// over the sample's atoms in fp64, then a fixed-order tree over the channels
// (block of 128 threads per sample; red is [D][128] shared doubles).
__device__ __forceinline__ void sample_energy(const Dev& d, int s, double* red) {
    const int D = d.D, H = d.H;
    const int64_t lo = d.atom_ptr[s], hi = d.atom_ptr[s + 1];
    const float* __restrict__ hL = d.h[d.L];
    double acc[kMaxHeads];
#pragma unroll
    for (int dd = 0; dd < kMaxHeads; ++dd) acc[dd] = 0.0;
    const int a = threadIdx.x;
    if (a < H) {
        float w[kMaxHeads];
#pragma unroll
        for (int dd = 0; dd < kMaxHeads; ++dd) w[dd] = dd < D ? d.we[a * D + dd] : 0.f;
        // 8 independent row loads in flight per iteration
        for (int64_t i0 = lo; i0 < hi; i0 += 8) {
            float hv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) hv[u] = i0 + u < hi ? __ldg(hL + (i0 + u) * H + a) : 0.f;
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int dd = 0; dd < kMaxHeads; ++dd)
                    if (dd < D) acc[dd] = fma(static_cast<double>(hv[u]), static_cast<double>(w[dd]), acc[dd]);
        }
    }
    // fixed-order reduction over the channels: butterfly within each warp, then
    // the 4 warp sums in order
#pragma unroll
    for (int dd = 0; dd < kMaxHeads; ++dd)
        if (dd < D)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[dd] += __shfl_xor_sync(0xffffffffu, acc[dd], o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int dd = 0; dd < kMaxHeads; ++dd)
            if (dd < D) red[dd * 4 + warp] = acc[dd];
    __syncthreads();
    if (threadIdx.x < D) {
        const double* r = red + threadIdx.x * 4;
        d.Epred[static_cast<int64_t>(s) * D + threadIdx.x] = ((r[0] + r[1]) + r[2]) + r[3];
    }
    __syncthreads();
}

// The train step's loss reads only the sample's own head: E_s^{d_s} alone.
__device__ __forceinline__ void sample_energy_own(const Dev& d, int s, int ds, double* red) {
    const int D = d.D, H = d.H;
    const int64_t lo = d.atom_ptr[s], hi = d.atom_ptr[s + 1];
    const float* __restrict__ hL = d.h[d.L];
    double acc = 0.0;
    const int a = threadIdx.x;
    if (a < H) {
        const double w = static_cast<double>(d.we[a * D + ds]);
        for (int64_t i0 = lo; i0 < hi; i0 += 8) {
            float hv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) hv[u] = i0 + u < hi ? __ldg(hL + (i0 + u) * H + a) : 0.f;
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = fma(static_cast<double>(hv[u]), w, acc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) d.Epred[static_cast<int64_t>(s) * D + ds] = ((red[0] + red[1]) + red[2]) + red[3];
    __syncthreads();
}

__global__ void __launch_bounds__(128) k_energy(Dev d) {
    pdl_enter();
    double* red = dyn_smem<double>();  // [D][128]
    const int B = d.hdr->B;
    for (int s = blockIdx.x; s < B; s += gridDim.x) sample_energy(d, s, red);
}

// ------------------------------------------------------------------ loss ---
// Eq. (5) with the per-rank denominators sum m_E, sum m_F (S/loss.cpp:175-212):
// block per sample (optionally computing its energies first) writes its energy
// and force terms and d(loss)/d(pred) for the selected head d_s only (every
// other channel is zeroed). The last block to finish sums the per-sample terms
// in index order (deterministic), publishes the rank's loss to the header and,
// as an fp32 hi/lo pair, into the allreduce payload after the gradients.
__global__ void __launch_bounds__(128) k_loss(Dev d, int with_energy, int full_gF) {
    pdl_enter();
    double* ered = dyn_smem<double>();  // [D][128] when with_energy
    __shared__ double red[128], red2[128];
    __shared__ bool last;
    const int B = d.hdr->B, D = d.D;
    const int me = d.hdr->me, mf = d.hdr->mf;
    const double we = me > 0 ? d.hdr->lambda_e / static_cast<double>(me) : 0.0;
    const double wf = mf > 0 ? d.hdr->lambda_f / static_cast<double>(mf) : 0.0;
    for (int s = blockIdx.x; s < B; s += gridDim.x) {
        const int ds = d.dsidx[s];
        if (with_energy) sample_energy_own(d, s, ds, ered);
        const int64_t lo = d.atom_ptr[s], hi = d.atom_ptr[s + 1];
        const bool em = d.emask[s], fm = d.fmask[s];
        const double ws = wf / static_cast<double>(hi - lo);
        double fsum = 0.0;
        for (int64_t a = lo + threadIdx.x; a < hi; a += 128) {
            float* g = d.gF + a * 3 * D;  // prediction-layout gradient: only for the API (lamm_loss_grad)
            if (full_gF)
                for (int q = 0; q < 3 * D; ++q) g[q] = 0.f;
            float4 gc = make_float4(0.f, 0.f, 0.f, 0.f);
            if (fm) {
                double df[3], sq = 0.0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    df[c] = static_cast<double>(d.F[(a * D + ds) * 3 + c]) - d.Fn[3 * a + c];
                    sq += df[c] * df[c];
                }
                const double dist = sqrt(sq);
                fsum += ws * dist;
                if (dist > 0.0) {
                    gc.x = static_cast<float>(ws * df[0] / dist);
                    gc.y = static_cast<float>(ws * df[1] / dist);
                    gc.z = static_cast<float>(ws * df[2] / dist);
                    if (full_gF) g[ds * 3] = gc.x, g[ds * 3 + 1] = gc.y, g[ds * 3 + 2] = gc.z;
                }
            }
            d.gFc[a] = gc;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = fsum;
        __syncthreads();
        if (threadIdx.x == 0) red[0] = ((red[0] + red[1]) + red[2]) + red[3];
        __syncthreads();
        if (threadIdx.x < D) {
            float ge = 0.f;
            if (threadIdx.x == ds && em) {
                const double diff = d.Epred[static_cast<int64_t>(s) * D + ds] - d.En[s];
                ge = diff > 0.0 ? static_cast<float>(we) : (diff < 0.0 ? static_cast<float>(-we) : 0.f);
            }
            d.gE[static_cast<int64_t>(s) * D + threadIdx.x] = ge;
        }
        if (threadIdx.x == 0) {
            double et = 0.0;
            if (em) et = we * fabs(d.Epred[static_cast<int64_t>(s) * D + ds] - d.En[s]);
            d.sample_terms[2 * s] = et;
            d.sample_terms[2 * s + 1] = fm ? red[0] : 0.0;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&d.hdr->done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double e = 0.0, f = 0.0;
    for (int s = threadIdx.x; s < B; s += 128) e += d.sample_terms[2 * s], f += d.sample_terms[2 * s + 1];
    red[threadIdx.x] = e, red2[threadIdx.x] = f;
    __syncthreads();
    for (int o = 64; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o], red2[threadIdx.x] += red2[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double tot = red[0] + red2[0];
        d.hdr->loss_energy = red[0];
        d.hdr->loss_force = red2[0];
        d.hdr->loss_total = tot;
        const float hi = static_cast<float>(tot);
        d.grads[d.NP] = hi;
        d.grads[d.NP + 1] = static_cast<float>(tot - static_cast<double>(hi));
        d.grads[d.NP + 2] = d.hdr->overflow ? 1.f : 0.f;
        d.grads[d.NP + 3] = 1.f;
        d.hdr->done_counter = 0;
    }
}

// ------------------------------------------------------------ evaluation ---
// trainer::evaluate (S/trainer.cpp:491-553) on the forward predictions: the
// sample's own head denormalized (S/loss.cpp:128-136), |E - E_label| / n and
// sum |F - F_label| / 3n per sample from the raw labels of the staged blob; the
// last block sums the per-sample terms in index order into the header
// (loss_energy, loss_force).
__global__ void __launch_bounds__(128) k_eval(Dev d) {
    pdl_enter();
    __shared__ double red[4];
    __shared__ bool last;
    const StepHeader& hd = *d.hdr;
    const char* base = reinterpret_cast<const char*>(d.hdr);
    const double* E = reinterpret_cast<const double*>(base + hd.off_E);
    const double* F = reinterpret_cast<const double*>(base + hd.off_F);
    const int B = hd.B, D = d.D;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = blockIdx.x; s < B; s += gridDim.x) {
        const int64_t lo = d.atom_ptr[s], hi = d.atom_ptr[s + 1];
        const double n = static_cast<double>(hi - lo);
        const int ds = d.dsidx[s];
        const bool em = d.emask[s], fm = d.fmask[s];
        if (threadIdx.x == 0) {
            double et = 0.0;
            if (em) {
                double e = d.Epred[static_cast<int64_t>(s) * D + ds];
                if (d.use_table) {
                    double refsum = 0.0;  // reference_sum, atoms in order
                    for (int64_t a = lo; a < hi; ++a)
                        if (d.rho_has[ds * 119 + d.Z[a]]) refsum = __dadd_rn(refsum, d.rho[ds * 119 + d.Z[a]]);
                    e = e * d.tstd[ds] + d.tmean[ds] + refsum;
                }
                et = fabs(e - E[s]) / n;
            }
            d.sample_terms[2 * s] = et;
        }
        double fsum = 0.0;
        if (fm) {
            const double fs = d.use_table ? d.tfstd[ds] : 1.0;
            for (int64_t a = lo + threadIdx.x; a < hi; a += blockDim.x)
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    fsum += fabs(static_cast<double>(d.F[(a * D + ds) * 3 + c]) * fs - F[3 * a + c]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
        if (lane == 0) red[warp] = fsum;
        __syncthreads();
        if (threadIdx.x == 0) d.sample_terms[2 * s + 1] = fm ? (((red[0] + red[1]) + red[2]) + red[3]) / (3.0 * n) : 0.0;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&d.hdr->done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double e = 0.0, f = 0.0;
    for (int s = threadIdx.x; s < B; s += blockDim.x) e += d.sample_terms[2 * s], f += d.sample_terms[2 * s + 1];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, o);
        f += __shfl_xor_sync(0xffffffffu, f, o);
    }
    __shared__ double re[4], rf[4];
    if (lane == 0) re[warp] = e, rf[warp] = f;
    __syncthreads();
    if (threadIdx.x == 0) {
        d.hdr->loss_energy = ((re[0] + re[1]) + re[2]) + re[3];
        d.hdr->loss_force = ((rf[0] + rf[1]) + rf[2]) + rf[3];
        d.hdr->done_counter = 0;
    }
}

// ------------------------------------------------------ embedding grad ---
// dE[Z_i - 1] += gh_i over the atoms after the layer-0 backward
// (S/model.cpp:421-424): CTA c sums a contiguous atom range per distinct-Z slot
// in shared memory (thread = channel, atoms in index order: deterministic) and
// writes one [nslots][H] partial; k_grad_reduce maps slots back to Z rows.
__global__ void __launch_bounds__(128) k_emb_grad(Dev d) {
    pdl_enter();
    float* acc = dyn_smem<float>();  // [kMaxZ][H]
    const int H = d.H, ns = d.hdr->nslots, N = d.hdr->N;
    const int a = threadIdx.x;
    for (int e = threadIdx.x; e < ns * H; e += blockDim.x) acc[e] = 0.f;
    __syncthreads();
    const int per = (N + gridDim.x - 1) / gridDim.x;
    const int i0 = min(N, static_cast<int>(blockIdx.x) * per), i1 = min(N, i0 + per);
    if (a < H) {
        for (int i = i0; i < i1; i += 8) {
            float v[8];
            int z[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const bool ok = i + u < i1;
                v[u] = ok ? __ldg(d.gh + static_cast<int64_t>(i + u) * H + a) : 0.f;
                z[u] = ok ? __ldg(d.zslot + i + u) : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[z[u] * H + a] += v[u];
        }
    }
    __syncthreads();
    float* part = d.part_emb + static_cast<int64_t>(blockIdx.x) * ns * H;
    for (int e = threadIdx.x; e < ns * H; e += blockDim.x) part[e] = acc[e];
}

// ------------------------------------------------------- grad reduction ---
struct Seg {
    int64_t dst;
    int32_t n, kind;  // kind 0: dense, 1: embedding rows through z_to_slot, 2: column-split
    const float* src;
    int32_t ncta, stride;
};
struct SegTable {
    int nseg;
    Seg s[2 * kMaxLayers + 4];
};

// grads[e] = sum over CTAs of the partials of the tensor that owns flat index e
// (for_each_tensor order). Block = 32 consecutive elements x 8 CTA-strided
// partial streams (coalesced loads, 8 independent sums per element), combined
// in a fixed order: deterministic for a fixed grid.
__global__ void __launch_bounds__(256) k_grad_reduce(Dev d, SegTable tab) {
    pdl_enter();
    __shared__ float red[8][33];
    const int H = d.H;
    const int ns = d.hdr->nslots;
    const int k = threadIdx.x & 31, g = threadIdx.x >> 5;
    for (int64_t e0 = static_cast<int64_t>(blockIdx.x) * 32; e0 < d.NP; e0 += static_cast<int64_t>(gridDim.x) * 32) {
        const int64_t e = e0 + k;
        float acc = 0.f;
        if (e < d.NP) {
            int q = 0;
            while (q + 1 < tab.nseg && e >= tab.s[q + 1].dst) ++q;
            const Seg& sg = tab.s[q];
            const int64_t off = e - sg.dst;
            // this thread's partial stream: first CTA c0, CTA step cs, element base + c * stride
            const float* base = nullptr;
            int c0 = g, cs = 8;
            int64_t stride = sg.stride;
            if (sg.kind == 1) {
                const int zrow = static_cast<int>(off / H), a = static_cast<int>(off % H);
                const int slot = d.z_to_slot[zrow + 1];
                if (slot >= 0) base = sg.src + slot * H + a;
                stride = static_cast<int64_t>(ns) * H;
            } else if (sg.kind == 2) {
                // column-split partials: CTA c holds columns [np*nc, np*nc+nc), np = c % (H/nc)
                const int nc = sg.stride / H, nsplit = H / nc;
                const int b = static_cast<int>(off / H), a = static_cast<int>(off % H), np = a / nc;
                base = sg.src + b * nc + (a - np * nc);
                c0 = np + nsplit * g;
                cs = 8 * nsplit;
            } else {
                base = sg.src + off;
            }
            if (base) {  // 4 loads in flight per step, summed in stream order
                int c = c0;
                for (; c + 3 * cs < sg.ncta; c += 4 * cs) {
                    const float v0 = __ldcg(base + c * stride), v1 = __ldcg(base + (c + cs) * stride);
                    const float v2 = __ldcg(base + (c + 2 * cs) * stride), v3 = __ldcg(base + (c + 3 * cs) * stride);
                    acc = (((acc + v0) + v1) + v2) + v3;
                }
                for (; c < sg.ncta; c += cs) acc += __ldcg(base + c * stride);
            }
        }
        red[g][k] = acc;
        __syncthreads();
        if (g == 0 && e < d.NP) {
            float s = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) s += red[q][k];
            d.grads[e] = s;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ optimizer ---
// Grid-wide barrier for a cooperative launch (all CTAs co-resident): arrival
// counter + generation word, the last arrival resets the counter and bumps the
// generation.
__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* vgen = gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// Mean over ranks (x 1/G as scale_params does), global norm (fp64, fixed-order
// tree over a fixed grid), non-finite check and clip factor, then
// RmsOptimizer::step with bit-exact fp64 arithmetic given the same gradient
// (S/trainer.cpp:37-53, 319-326); refreshes the fp32 working copy and tanh(E)
// for layer 0's gathers. Every CTA reduces the per-CTA norms itself, so no
// second barrier is needed before the update. Returns the step status.
template <class OnParam>
__device__ __forceinline__ int opt_update(const Dev& d, int G, double inv_g, double clip, double lr, double decay,
                                          double eps, unsigned int* bar, OnParam on_param) {
    __shared__ double red[256];
    double s = 0.0;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < d.NP;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double g = __dmul_rn(d.g64_in ? d.g64_in[e] : static_cast<double>(d.grads[e]), inv_g);
        s += g * g;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) d.block_scratch[blockIdx.x] = red[0];
    grid_barrier(bar, bar + 32);
    red[threadIdx.x] = threadIdx.x < gridDim.x ? d.block_scratch[threadIdx.x] : 0.0;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    const double gn = sqrt(red[0]);
    double loss = 0.0;
    if (!d.g64_in)
        loss = (static_cast<double>(d.grads[d.NP]) + static_cast<double>(d.grads[d.NP + 1])) / static_cast<double>(G);
    else if (d.g64_loss)
        loss = (d.g64_in[d.NP] + d.g64_in[d.NP + 1]) / static_cast<double>(G);
    const bool overflow = !d.g64_in && d.grads[d.NP + 2] > 0.f;
    const int status = overflow ? 2 : ((!isfinite(loss) || !isfinite(gn)) ? 1 : 0);
    const double cs = (clip > 0.0 && gn > clip) ? clip / gn : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        d.hdr->grad_norm = gn;
        d.hdr->global_loss = loss;
        d.hdr->status = status;
        d.hdr->clip_scale = cs;
        if (status != 0 && !d.g64_in) atomicAdd(d.anomaly, 1u);
    }
    if (status != 0) return status;
    const int64_t emb_n = static_cast<int64_t>(kMaxZ) * d.H;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < d.NP;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double g = __dmul_rn(d.g64_in ? d.g64_in[e] : static_cast<double>(d.grads[e]), inv_g);
        if (cs != 0.0) g = __dmul_rn(g, cs);
        const double v = __dadd_rn(__dmul_rn(decay, d.v64[e]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, decay), g), g));
        const double p = __dsub_rn(d.p64[e], __ddiv_rn(__dmul_rn(lr, g), __dadd_rn(__dsqrt_rn(v), eps)));
        d.v64[e] = v;
        d.p64[e] = p;
        const float pf = static_cast<float>(p);
        d.p32[e] = pf;
        if (e < emb_n) d.tanh_emb_w[e] = tanhf(pf);
        on_param(e, pf);
    }
    return status;
}

// Simulated workers on one device (S/trainer.cpp:262-319: G device-batches in
// worker order, gradients summed before one optimizer step): worker g's packed
// gradient and loss terms added to the fp64 accumulator in worker order.
__global__ void __launch_bounds__(256) k_grad_accum(Dev d, int first) {
    pdl_enter();
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < d.NP + 2;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = static_cast<double>(d.grads[e]);
        d.g64_acc[e] = first ? v : d.g64_acc[e] + v;
    }
}

// fp64 master -> fp32 working copy (+ tanh(E)) after a host parameter upload.
__global__ void __launch_bounds__(256) k_params_cast(Dev d) {
    pdl_enter();
    const int64_t emb_n = static_cast<int64_t>(kMaxZ) * d.H;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < d.NP;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float pf = static_cast<float>(d.p64[e]);
        d.p32[e] = pf;
        if (e < emb_n) d.tanh_emb_w[e] = tanhf(pf);
    }
}

}  // namespace lamm_b200
