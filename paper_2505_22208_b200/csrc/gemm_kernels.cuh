// gemm_kernels.cuh - the per-atom dense contractions of the step on tcgen05
// tensor cores (3xTF32, fp32-accurate), accumulators in TMEM.
//
//   k_node_gemm mode 0 (update, S/model.cpp:93-102):   Y = mu_l W_u^T   (M = 128 atoms, N = H, K = H)
//               epilogue h_{l+1} = h_l + Y, t_{l+1} = tanh h_{l+1}; last layer also
//               e_i = W_e^T h^L_i and A_i = W_fh[0:H]^T t^L_i   (S/model.cpp:208-218, 232-240)
//   k_node_gemm mode 1 (S/model.cpp:380-390):          gm = (gh W_u) (.) (1 - mu^2)
//   k_dwu              (S/model.cpp:381-383):          dW_u = gh^T mu, split-K over atoms
//                                                       (one per-CTA partial, summed by k_grad_reduce)
//
// One 128-thread CTA per SM, persistent over 128-atom tiles. The weight matrix
// stays resident in shared memory as tf32 hi/lo K-major tiles; activations are
// staged K-chunk by K-chunk (32 wide, double buffered) into hi/lo tiles by the
// threads, then thread 0 issues the tcgen05.mma chain (12 per chunk) and
// commits to an mbarrier; the epilogue reads the accumulator with tcgen05.ld
// (thread = TMEM lane = one atom row).
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"
#include "edge_kernels.cuh"
#include "kernels.cuh"
#include "umma.cuh"

namespace lamm_b200 {

constexpr int kGemmM = 128;      // atoms per tile (TMEM lanes)
constexpr int kGemmKC = 32;      // K chunk of the staged activations
constexpr int kGemmMaxHeads = 16;

template <int H>
struct NodeGemmSmem {
    static constexpr size_t b_floats = 2 * H * H;                    // W hi | lo
    static constexpr size_t a_floats = 2 * 2 * kGemmM * kGemmKC;     // 2 stages x (hi | lo)
    static constexpr size_t heads_floats = 2 * H * kGemmMaxHeads;    // W_e | W_fh[0:H] (last layer)
    static constexpr size_t bytes = 4 * (b_floats + a_floats + heads_floats) + 64;
};

// Stages rows [base, base+128) x cols [k0, k0+KC) of a row-major [N][H] fp32
// array into hi/lo K-major canonical tiles (rows >= N are zero).
template <int H>
__device__ __forceinline__ void stage_rows(const float* __restrict__ src, int N, int base, int k0, float* Ahi,
                                           float* Alo) {
    constexpr int Q = kGemmKC / 4;
    for (int q = threadIdx.x; q < kGemmM * Q; q += blockDim.x) {
        const int m = q / Q, k4 = q % Q, atom = base + m;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (atom < N) v = *reinterpret_cast<const float4*>(src + static_cast<int64_t>(atom) * H + k0 + 4 * k4);
        float4 hi, lo;
        umma::split_tf32(v.x, hi.x, lo.x);
        umma::split_tf32(v.y, hi.y, lo.y);
        umma::split_tf32(v.z, hi.z, lo.z);
        umma::split_tf32(v.w, hi.w, lo.w);
        const int o = umma::kidx(m, 4 * k4, kGemmKC);
        *reinterpret_cast<float4*>(Ahi + o) = hi;
        *reinterpret_cast<float4*>(Alo + o) = lo;
    }
}

template <int H>
__global__ void __launch_bounds__(128, 1) k_node_gemm(Dev d, int l, int mode, int last) {
    static_assert(H % kGemmKC == 0 && H >= 32 && H <= 128, "node GEMM supports H in {32, 64, 128}");
    constexpr int NKC = H / kGemmKC;
    float* sm = dyn_smem<float>();
    float* Bhi = sm;
    float* Blo = Bhi + H * H;
    float* Ast = Blo + H * H;
    float* We = Ast + 2 * 2 * kGemmM * kGemmKC;
    float* Wa = We + H * kGemmMaxHeads;
    uint64_t* bar = reinterpret_cast<uint64_t*>(Wa + H * kGemmMaxHeads);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int D = d.D;
    if (warp == 0) umma::tmem_alloc(tslot, H);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    const float* __restrict__ wu = d.wu[l];
    for (int idx = tid; idx < H * H; idx += blockDim.x) {
        const int n = idx / H, k = idx % H;  // B[n][k]: update W_u[n][k]; gm W_u[k][n]
        float hi, lo;
        umma::split_tf32(mode == 0 ? wu[idx] : wu[k * H + n], hi, lo);
        Bhi[umma::kidx(n, k, H)] = hi;
        Blo[umma::kidx(n, k, H)] = lo;
    }
    if (last)
        for (int idx = tid; idx < H * D; idx += blockDim.x) We[idx] = d.we[idx], Wa[idx] = d.wfh[idx];
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = *tslot;
    const uint32_t idesc = umma::idesc_tf32(kGemmM, H);
    const int N = d.hdr->N;
    const int ntiles = (N + kGemmM - 1) / kGemmM;
    const float* __restrict__ src = mode == 0 ? d.mu[l] : d.gh;
    int chunk = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int base = tile * kGemmM;
        for (int kc = 0; kc < NKC; ++kc, ++chunk) {
            const int st = chunk & 1;
            if (chunk >= 2) mbar_wait(&bar[st], ((chunk - 2) >> 1) & 1);  // MMAs that read this stage are done
            float* Ahi = Ast + st * 2 * kGemmM * kGemmKC;
            float* Alo = Ahi + kGemmM * kGemmKC;
            stage_rows<H>(src, N, base, kc * kGemmKC, Ahi, Alo);
            umma::fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                umma::fence_after();
#pragma unroll
                for (int s = 0; s < kGemmKC / 8; ++s) {
                    const int sg = kc * (kGemmKC / 8) + s;
                    umma::mma3(tbase, umma::kdesc(Ahi, s, kGemmKC), umma::kdesc(Alo, s, kGemmKC),
                               umma::kdesc(Bhi, sg, H), umma::kdesc(Blo, sg, H), idesc, (kc | s) ? 1u : 0u);
                }
                umma::commit(&bar[st]);
            }
        }
        const int lc = chunk - 1;
        mbar_wait(&bar[lc & 1], (lc >> 1) & 1);
        umma::fence_after();
        const int row = warp * 32 + lane, atom = base + row;
        const bool live = atom < N;
        float eacc[kGemmMaxHeads], aacc[kGemmMaxHeads];
#pragma unroll
        for (int q = 0; q < kGemmMaxHeads; ++q) eacc[q] = aacc[q] = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < H; c0 += 16) {
            float v[16];
            umma::ld16(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            if (!live) continue;
            if (mode == 0) {
                const float* hp = l == 0 ? d.emb + static_cast<int64_t>(__ldg(d.Z + atom) - 1) * H
                                         : d.h[l] + static_cast<int64_t>(atom) * H;
                float hn[16], tn[16];
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    const float4 hv = *reinterpret_cast<const float4*>(hp + c0 + q);
                    hn[q] = hv.x + v[q], hn[q + 1] = hv.y + v[q + 1], hn[q + 2] = hv.z + v[q + 2],
                    hn[q + 3] = hv.w + v[q + 3];
                }
#pragma unroll
                for (int q = 0; q < 16; ++q) tn[q] = tanhf(hn[q]);
                float* ho = d.h[l + 1] + static_cast<int64_t>(atom) * H + c0;
                float* to = d.t[l + 1] + static_cast<int64_t>(atom) * H + c0;
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    *reinterpret_cast<float4*>(ho + q) = make_float4(hn[q], hn[q + 1], hn[q + 2], hn[q + 3]);
                    *reinterpret_cast<float4*>(to + q) = make_float4(tn[q], tn[q + 1], tn[q + 2], tn[q + 3]);
                }
                if (last) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const float* we = We + (c0 + q) * D;
                        const float* wa = Wa + (c0 + q) * D;
#pragma unroll
                        for (int dd = 0; dd < kGemmMaxHeads; ++dd)
                            if (dd < D) eacc[dd] = fmaf(hn[q], we[dd], eacc[dd]), aacc[dd] = fmaf(tn[q], wa[dd], aacc[dd]);
                    }
                }
            } else {
                const float* mp = d.mu[l] + static_cast<int64_t>(atom) * H + c0;
                float* go = d.gm + static_cast<int64_t>(atom) * H + c0;
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    const float4 m4 = *reinterpret_cast<const float4*>(mp + q);
                    *reinterpret_cast<float4*>(go + q) =
                        make_float4(v[q] * (1.f - m4.x * m4.x), v[q + 1] * (1.f - m4.y * m4.y),
                                    v[q + 2] * (1.f - m4.z * m4.z), v[q + 3] * (1.f - m4.w * m4.w));
                }
            }
        }
        if (mode == 0 && last && live) {
#pragma unroll
            for (int dd = 0; dd < kGemmMaxHeads; ++dd)
                if (dd < D) {
                    d.e_atom[static_cast<int64_t>(atom) * D + dd] = eacc[dd];
                    d.A[static_cast<int64_t>(atom) * D + dd] = aacc[dd];
                }
        }
        umma::fence_before();
        __syncthreads();  // accumulator drained before the next tile's first MMA
        umma::fence_after();
    }
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tbase, H);
}

template <int H>
struct DwuSmem {
    static constexpr size_t stage_floats = 4 * kGemmM * kGemmKC;  // A hi|lo, B hi|lo
    static constexpr size_t bytes = 4 * 2 * stage_floats + 64;
};

// dW_u[b][a] = sum_atoms gh[atom][b] mu[atom][a]: M = b (rows >= H zero), N = H,
// K = atoms in 32-atom chunks; CTA c reduces a contiguous chunk range.
template <int H>
__global__ void __launch_bounds__(128, 1) k_dwu(Dev d, int l) {
    constexpr int Q = H / 4;
    float* sm = dyn_smem<float>();
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * DwuSmem<H>::stage_floats);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) umma::tmem_alloc(tslot, H);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    // rows H..127 of the A tiles stay zero
    for (int e = tid; e < 2 * DwuSmem<H>::stage_floats; e += blockDim.x) sm[e] = 0.f;
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = *tslot;
    const uint32_t idesc = umma::idesc_tf32(kGemmM, H);
    const int N = d.hdr->N;
    const int nch = (N + kGemmKC - 1) / kGemmKC;
    const int c0 = static_cast<int>((static_cast<int64_t>(nch) * blockIdx.x) / gridDim.x);
    const int c1 = static_cast<int>((static_cast<int64_t>(nch) * (blockIdx.x + 1)) / gridDim.x);
    const float* __restrict__ gh = d.gh;
    const float* __restrict__ mu = d.mu[l];
    int q = 0;
    for (int ch = c0; ch < c1; ++ch, ++q) {
        const int st = q & 1;
        if (q >= 2) mbar_wait(&bar[st], ((q - 2) >> 1) & 1);
        float* Ahi = sm + st * DwuSmem<H>::stage_floats;
        float* Alo = Ahi + kGemmM * kGemmKC;
        float* Bhi = Alo + kGemmM * kGemmKC;
        float* Blo = Bhi + kGemmM * kGemmKC;
        for (int it = tid; it < kGemmKC * Q; it += blockDim.x) {
            const int al = it / Q, c4 = it % Q, atom = ch * kGemmKC + al;
            float4 g = make_float4(0.f, 0.f, 0.f, 0.f), m = g;
            if (atom < N) {
                g = *reinterpret_cast<const float4*>(gh + static_cast<int64_t>(atom) * H + 4 * c4);
                m = *reinterpret_cast<const float4*>(mu + static_cast<int64_t>(atom) * H + 4 * c4);
            }
            const float gv[4] = {g.x, g.y, g.z, g.w}, mv[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int o = umma::kidx(4 * c4 + r, al, kGemmKC);
                umma::split_tf32(gv[r], Ahi[o], Alo[o]);
                umma::split_tf32(mv[r], Bhi[o], Blo[o]);
            }
        }
        umma::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            umma::fence_after();
#pragma unroll
            for (int s = 0; s < kGemmKC / 8; ++s)
                umma::mma3(tbase, umma::kdesc(Ahi, s, kGemmKC), umma::kdesc(Alo, s, kGemmKC),
                           umma::kdesc(Bhi, s, kGemmKC), umma::kdesc(Blo, s, kGemmKC), idesc,
                           (q | s) ? 1u : 0u);
            umma::commit(&bar[st]);
        }
    }
    if (q > 0) {
        mbar_wait(&bar[(q - 1) & 1], ((q - 1) >> 1) & 1);
        umma::fence_after();
    }
    const int row = warp * 32 + lane;
    float* part = d.part_wu[l] + static_cast<int64_t>(blockIdx.x) * H * H;
#pragma unroll 1
    for (int c = 0; c < H; c += 16) {
        float v[16];
        umma::ld16(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
        if (row < H)
#pragma unroll
            for (int k = 0; k < 16; k += 4)
                *reinterpret_cast<float4*>(part + row * H + c + k) =
                    q > 0 ? make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tbase, H);
}

}  // namespace lamm_b200
