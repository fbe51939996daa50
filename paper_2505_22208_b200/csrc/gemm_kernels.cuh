// gemm_kernels.cuh - the per-atom dense contractions of the step on tcgen05
// tensor cores (3xTF32, fp32-accurate), accumulators in TMEM.
//
//   k_message_update (train step, H = 128; S/model.cpp:78-102): the message walk of
//               the CTA's edge partitions, then the update GEMM of the CTA's own atoms
//               Y = mu_l W_u^T (M = 128 atom rows per tile, two 64-column W_u blocks
//               by TMA, 48 MMAs each), epilogue h_{l+1} = h_l + Y, t_{l+1} = tanh
//   k_bwd_gemm  (train step, H = 128; S/model.cpp:380-390): gm = (gh W_u) (.) (1 - mu^2)
//               fused with dW_u = gh^T mu (per-CTA partial, summed by k_grad_reduce)
//   k_node_gemm mode 0 / 1 and k_dwu: the same contractions as separate kernels
//               (forward / backward entry points and H != 128)
//
// Geometry: one CTA per SM, 512 threads (256 for H = 32) = 4 threads per TMEM lane:
// warps w, w + 4, w + 8, w + 12 share lanes 32 (w % 4) .. + 31 and split the output
// columns. Activation tiles arrive by TMA (SWIZZLE_128B boxes, the raw fp32 values
// as the tf32 hi operand, lo = x - trunc_tf32(x) split in place by the threads);
// weight blocks are K-major canonical hi/lo tiles packed by k_pack_weights / k_opt
// and fetched with one bulk copy, before the dependency wait where the weights are
// at least two kernels old. Thread 0 issues the MMA chain (3 per k-step of 8) and
// commits to an mbarrier; the epilogue reads the accumulator with tcgen05.ld.
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"
#include "edge_kernels.cuh"
#include "kernels.cuh"
#include "umma.cuh"

namespace lamm_b200 {

constexpr int kGemmM = 128;      // atoms per tile (TMEM lanes)
constexpr int kGemmKC = 32;      // K chunk of the staged activations

// Column split of a node-GEMM tile: for H = 128 two CTAs share a 128-atom
// tile (64 output columns each) so small batches still fill the GPU.
template <int H>
struct NodeGemmCfg {
    static constexpr int NS = H == 128 ? 2 : 1;
    static constexpr int NC = H / NS;                       // output columns per CTA tile
    static constexpr int NT = H == 32 ? 256 : 512;          // k_node_gemm threads (4 per TMEM lane)
    static constexpr size_t a_floats = 2 * kGemmM * H;      // activation tile hi | lo (full K)
    static constexpr size_t b_floats = 2 * NC * H;          // weight rows [NC][H] hi | lo
    static constexpr size_t bytes = 4 * (a_floats + b_floats) + 64 + 1024;  // + barriers, alignment slack
};
template <int H>
using NodeGemmSmem = NodeGemmCfg<H>;

// Weight operands of the node GEMMs, packed once per parameter update by
// k_pack_weights: per layer [4][H*H] = {W_u hi, W_u lo, W_u^T hi, W_u^T lo}.
// Each is split into NS row blocks of NC rows, every block a K-major canonical
// [NC][H] tile (B[n][k] = W_u[n][k] for the update, W_u[k][n] for gm), hi and
// lo blocks adjacent, so a CTA fetches its operand with one TMA bulk copy.
template <int H>
__device__ __forceinline__ void pack_weights(const Dev& d) {
    constexpr int NC = NodeGemmCfg<H>::NC;
    const int64_t per = static_cast<int64_t>(H) * H;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < d.L * per;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int l = static_cast<int>(e / per), idx = static_cast<int>(e % per);
        const int n = idx / H, k = idx % H;
        const float* wu = d.wu[l];
        const int blk = n / NC, o = umma::kidx(n % NC, k, H);
        // layout per layer and mode: [block][hi | lo][NC*H]
        float* upd = d.wpack + 4 * per * l + static_cast<int64_t>(blk) * 2 * NC * H;
        float* gm = upd + 2 * per;
        umma::split_tf32(wu[idx], upd[o], upd[NC * H + o]);
        umma::split_tf32(wu[k * H + n], gm[o], gm[NC * H + o]);
    }
}

template <int H>
__global__ void __launch_bounds__(256) k_pack_weights(Dev d) {
    pdl_enter();
    pack_weights<H>(d);
}

// The optimizer tail of the step as ONE cooperative kernel (grid <= 256 CTAs of
// 256 threads, all co-resident): norm -> barrier -> clip + RMS update, each
// updated W_u element scattered straight into both tensor-core weight packs
// (its W_u and W_u^T positions), so no second grid barrier is needed.
template <int H>
__global__ void __launch_bounds__(256) k_opt(Dev d, int G, double inv_g, double clip, double lr, double decay,
                                             double eps) {
    pdl_enter();
    constexpr int NC = NodeGemmCfg<H>::NC;
    const int64_t per = static_cast<int64_t>(H) * H;
    const int64_t wu0 = static_cast<int64_t>(kMaxZ) * H + static_cast<int64_t>(d.L) * H * d.K;  // W_u[0] offset
    unsigned int* bar = d.anomaly + 16;
    opt_update(d, G, inv_g, clip, lr, decay, eps, bar, [&](int64_t e, float w) {
        const int64_t r = e - wu0;
        if (r < 0 || r >= d.L * per) return;
        const int l = static_cast<int>(r / per), idx = static_cast<int>(r % per);
        const int n = idx / H, k = idx % H;  // W_u[n][k]: output n, input k
        float* upd = d.wpack + 4 * per * l;
        float* gm = upd + 2 * per;
        // update operand B[n][k] = W_u[n][k]; backward operand B'[k][n] = W_u[n][k]
        float* ub = upd + static_cast<int64_t>(n / NC) * 2 * NC * H;
        float* gb = gm + static_cast<int64_t>(k / NC) * 2 * NC * H;
        const int ou = umma::kidx(n % NC, k, H), og = umma::kidx(k % NC, n, H);
        umma::split_tf32(w, ub[ou], ub[NC * H + ou]);
        umma::split_tf32(w, gb[og], gb[NC * H + og]);
    });
}

// One tile = 128 atoms x NC output columns, K = H, NT threads (512; 256 at H = 32):
// the activation tile arrives by TMA in 32-column SWIZZLE_128B boxes (one barrier
// each; the threads split box kb into hi/lo while the tensor core runs box kb - 1),
// the weight block by one bulk copy, 3*H/8 MMAs accumulate into TMEM, and the
// epilogue inputs (residual / mu) are prefetched while the tensor core runs.
// The NT/32 warps share TMEM lanes 32*(w%4).. in groups of four and split the NC columns.
template <int H>
__global__ void __launch_bounds__(NodeGemmCfg<H>::NT, 1) k_node_gemm(Dev d, int l, int mode, const __grid_constant__ CUtensorMap amap,
                                                      const __grid_constant__ CUtensorMap omap0,
                                                      const __grid_constant__ CUtensorMap omap1) {
    using Cfg = NodeGemmCfg<H>;
    constexpr int NS = Cfg::NS, NC = Cfg::NC, NT = Cfg::NT, CW = NC / (NT / 128);  // columns per thread
    constexpr int KB = H / 32;                               // 32-column activation boxes (TMA, SWIZZLE_128B)
    constexpr bool kTmaOut = CW == 16 || CW == 32;  // epilogue through shared memory + TMA stores
    static_assert(CW % 16 == 0, "epilogue reads 16 columns at a time");
    extern __shared__ __align__(1024) unsigned char node_gemm_smem[];
    float* sm = reinterpret_cast<float*>(node_gemm_smem + ((1024u - (smem_u32(node_gemm_smem) & 1023u)) & 1023u));
    float* Ahi = sm;  // the raw activation tile (TMA, SWIZZLE_128B): the tf32 "hi" operand as is
    float* Alo = Ahi + kGemmM * H;
    float* Bhi = Alo + kGemmM * H;
    // barriers: [0] weights TMA, [1] MMA done, [2, 2 + KB) activation boxes
    uint64_t* bar = reinterpret_cast<uint64_t*>(Bhi + Cfg::b_floats);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2 + KB);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quad = warp & 3, part = warp >> 2;  // TMEM lane quarter, column part
    constexpr uint32_t kCols = NC < 32 ? 32 : NC;
    if (warp == 0) umma::tmem_alloc(tslot, kCols);
    if (tid == 0) {
        for (int b = 0; b < 2 + KB; ++b) mbar_init(&bar[b], 1);
        mbar_fence_init();
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = *tslot;
    const uint32_t idesc = umma::idesc_tf32(kGemmM, NC);
    const int N = d.hdr->N;  // from the staged upload, not from the previous kernel
    const int ntiles = (N + kGemmM - 1) / kGemmM * NS;
    uint32_t wphase = 0, mphase = 0, aphase = 0;
    int loaded_np = -1;
    bool w_pending = false;
    auto fetch_weights = [&](int np) {  // weight block of a column split (TMA), packed by the last optimizer step
        if (tid == 0) {
            const float* wsrc =
                d.wpack + static_cast<int64_t>(4 * l + 2 * mode) * H * H + static_cast<int64_t>(np) * 2 * NC * H;
            mbar_expect_tx(&bar[0], static_cast<uint32_t>(Cfg::b_floats * 4));
            bulk_g2s(Bhi, wsrc, static_cast<uint32_t>(Cfg::b_floats * 4), &bar[0]);
        }
        loaded_np = np;
        w_pending = true;
    };
    if (static_cast<int>(blockIdx.x) < ntiles) fetch_weights(blockIdx.x % NS);  // overlaps the previous kernel
    pdl_enter();
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int at = tile / NS, np = tile % NS, base = at * kGemmM;
        if (np != loaded_np) fetch_weights(np);
        // the activation tile (mu_l or gh rows base..base+127, all H columns) by TMA
        // in KB SWIZZLE_128B boxes, one barrier each; rows past the batch are never stored
        if (tid == 0) {
            if constexpr (kTmaOut) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // last tile's stores
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                mbar_expect_tx(&bar[2 + kb], static_cast<uint32_t>(kGemmM * 32 * 4));
                umma::tma_load_2d(Ahi + kb * kGemmM * 32, &amap, kb * 32, base, &bar[2 + kb]);
            }
        }
        // per box as it lands: lo = x - trunc_tf32(x) at the same swizzled positions,
        // then its 4 k-steps (3 MMAs each) — the tensor core works on box kb while
        // the threads split box kb + 1
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&bar[2 + kb], aphase);
            constexpr int IT = kGemmM * 32 / 4 / NT;
#pragma unroll
            for (int it = 0; it < IT; ++it) {
                const int c = kb * kGemmM * 8 + tid + NT * it;
                const float4 x = *reinterpret_cast<const float4*>(Ahi + 4 * c);
                *reinterpret_cast<float4*>(Alo + 4 * c) =
                    make_float4(umma::tf32_trunc_lo(x.x), umma::tf32_trunc_lo(x.y), umma::tf32_trunc_lo(x.z),
                                umma::tf32_trunc_lo(x.w));
            }
            umma::fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                if (kb == 0 && w_pending) mbar_wait(&bar[0], wphase);
                umma::fence_after();
                const float* Blo = Bhi + NC * H;
#pragma unroll
                for (int s = 4 * kb; s < 4 * kb + 4; ++s)
                    umma::mma3(tbase, umma::sw128_kdesc(Ahi, s, kGemmM), umma::sw128_kdesc(Alo, s, kGemmM),
                               umma::kdesc(Bhi, s, H), umma::kdesc(Blo, s, H), idesc, s ? 1u : 0u);
                if (kb == KB - 1) umma::commit(&bar[1]);
            }
        }
        aphase ^= 1u;
        if (w_pending) wphase ^= 1u, w_pending = false;
        // epilogue inputs for this thread's row/columns, fetched while the MMAs run
        const int row = quad * 32 + lane, atom = base + row, c0 = np * NC + part * CW;
        const bool live = atom < N;
        float pre[CW];
#pragma unroll
        for (int q = 0; q < CW; ++q) pre[q] = 0.f;
        if (live) {
            const float* p = mode == 0 ? (l == 0 ? d.emb + static_cast<int64_t>(__ldg(d.Z + atom) - 1) * H
                                                 : d.h[l] + static_cast<int64_t>(atom) * H)
                                       : d.mu[l] + static_cast<int64_t>(atom) * H;
#pragma unroll
            for (int q = 0; q < CW; q += 4) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(p + c0 + q));
                pre[q] = x.x, pre[q + 1] = x.y, pre[q + 2] = x.z, pre[q + 3] = x.w;
            }
        }
        mbar_wait(&bar[1], mphase);
        mphase ^= 1u;
        umma::fence_after();
        if constexpr (kTmaOut) {
            // outputs as SWIZZLE_128B boxes [128 rows][32 columns] in the (now free)
            // activation tiles: box (array, b) = Ahi + (array * NC/32 + b) * 4096 holds tile
            // columns [32 b, 32 b + 32); thread row r writes its 16-byte chunk q at chunk
            // position q ^ (r % 8)
            const int cb = part * CW;  // first tile column of this thread
            float* ob = Ahi + (cb / 32) * kGemmM * 32 + row * 32;
#pragma unroll
            for (int cc = 0; cc < CW; cc += 16) {
                float v[16];
                umma::ld16(tbase + (static_cast<uint32_t>(quad * 32) << 16) + cb + cc, v);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const int q = (cb % 32 + cc) / 4 + q4, pos = (q ^ (row & 7)) * 4;
                    float4 a, b;
                    if (mode == 0) {
                        float hn[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) hn[e] = pre[cc + 4 * q4 + e] + v[4 * q4 + e];
                        a = make_float4(hn[0], hn[1], hn[2], hn[3]);
                        b = make_float4(tanhf(hn[0]), tanhf(hn[1]), tanhf(hn[2]), tanhf(hn[3]));
                    } else {
                        float g[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float m = pre[cc + 4 * q4 + e];
                            g[e] = v[4 * q4 + e] * (1.f - m * m);
                        }
                        a = b = make_float4(g[0], g[1], g[2], g[3]);
                    }
                    *reinterpret_cast<float4*>(ob + pos) = a;
                    if (mode == 0) *reinterpret_cast<float4*>(ob + (NC / 32) * kGemmM * 32 + pos) = b;
                }
            }
            umma::fence_proxy_async();  // generic-proxy writes -> visible to the TMA engine
            umma::fence_before();
            __syncthreads();
            if (tid == 0) {
                const int narr = mode == 0 ? 2 : 1;
                for (int arr = 0; arr < narr; ++arr)
                    for (int hf = 0; hf < NC / 32; ++hf)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                reinterpret_cast<uint64_t>(arr == 0 ? &omap0 : &omap1)),
                            "r"(np * NC + hf * 32), "r"(base), "r"(smem_u32(Ahi + (arr * (NC / 32) + hf) * kGemmM * 32))
                            : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            umma::fence_after();
        } else {
#pragma unroll
        for (int cc = 0; cc < CW; cc += 16) {
            float v[16];
            umma::ld16(tbase + (static_cast<uint32_t>(quad * 32) << 16) + part * CW + cc, v);
            if (!live) continue;
            if (mode == 0) {
                float hn[16], tn[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) hn[q] = pre[cc + q] + v[q], tn[q] = tanhf(hn[q]);
                float* ho = d.h[l + 1] + static_cast<int64_t>(atom) * H + c0 + cc;
                float* to = d.t[l + 1] + static_cast<int64_t>(atom) * H + c0 + cc;
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    *reinterpret_cast<float4*>(ho + q) = make_float4(hn[q], hn[q + 1], hn[q + 2], hn[q + 3]);
                    *reinterpret_cast<float4*>(to + q) = make_float4(tn[q], tn[q + 1], tn[q + 2], tn[q + 3]);
                }
            } else {
                float* go = d.gm + static_cast<int64_t>(atom) * H + c0 + cc;
#pragma unroll
                for (int q = 0; q < 16; q += 4)
                    *reinterpret_cast<float4*>(go + q) =
                        make_float4(v[q] * (1.f - pre[cc + q] * pre[cc + q]),
                                    v[q + 1] * (1.f - pre[cc + q + 1] * pre[cc + q + 1]),
                                    v[q + 2] * (1.f - pre[cc + q + 2] * pre[cc + q + 2]),
                                    v[q + 3] * (1.f - pre[cc + q + 3] * pre[cc + q + 3]));
            }
        }
        umma::fence_before();
        __syncthreads();  // accumulator and activation tile drained before the next tile
        umma::fence_after();
        }
    }
    if constexpr (kTmaOut)  // the stores have read shared memory (grid completion publishes the writes)
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tbase, kCols);
}

// ------------------------------------------------- message + update, fused --
// One encoder layer in ONE kernel (H = 128, S/model.cpp:78-102): the message walk
// of k_edge_message over the CTA's 12 edge partitions, then the update GEMM
//   h_{l+1} = h_l + mu W_u^T,  t_{l+1} = tanh(h_{l+1})
// for the CTA's OWN atoms - the rows its partitions cover, [a0, a1), contiguous
// and disjoint between CTAs - on tcgen05 (3xTF32, TMEM accumulator). No grid-wide
// dependency separates the two phases: every mu row the GEMM reads was written by
// this CTA's walk (visible after the CTA barrier), so the update needs neither its
// own launch nor a round trip through a dependency wait. Per 128-row tile:
//   A = the mu rows as a SWIZZLE_128B K-major tile (raw fp32 = the tf32 hi operand,
//       lo = x - trunc_tf32(x)) written by the threads into the walk's (dead) stage
//       region; B = a 64-column block of W_u (hi | lo, k_pack_weights' layout) by
//       one bulk copy - block 0 prefetched before the walk, block 1 once MMA 0 has
//       read block 0; accumulators in TMEM columns [0, 64) and [64, 128) of the
//       walk's allocation; epilogue: thread = (TMEM lane quarter, 16-column part).
template <int K>
struct MsgUpdSmem {
    static constexpr size_t a_bytes = 4 * 2 * kGemmM * 128;      // A hi | lo
    static constexpr size_t b_bytes = 4 * 2 * 64 * 128;          // one 64-column W_u block, hi | lo
    static constexpr size_t walk = EdgeSmem<K, kMsgGroups, kMsgChunk>::extra_offset + 4 * 2 * 128 * K;  // + W_f tiles
    static constexpr size_t b_off = ((walk > a_bytes + 1024 ? walk : a_bytes + 1024) + 127) / 128 * 128;
    static constexpr size_t bar_off = b_off + b_bytes;
    static constexpr size_t bytes = bar_off + 64;
};

template <int K, bool kZ>
__global__ void __launch_bounds__(kMsgGroups * 128, 1) k_message_update(Dev d, int l) {
    constexpr int H = 128, NC = 64;
    extern __shared__ __align__(128) unsigned char lamm_edge_smem[];
    EdgeCta<H, K, kMsgGroups, kMsgChunk> c = edge_prologue<H, K, kMsgGroups, kMsgChunk>(d, kZ);
    using Sm = MsgUpdSmem<K>;
    float* Bw = reinterpret_cast<float*>(lamm_edge_smem + Sm::b_off);
    uint64_t* gb = reinterpret_cast<uint64_t*>(lamm_edge_smem + Sm::bar_off);  // [0] weights, [1..2] MMA
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int b = 0; b < 3; ++b) mbar_init(&gb[b], 1);
        mbar_fence_init();
    }
    float* Wh = reinterpret_cast<float*>(c.extra);
    const FilterTc ft = filter_setup<H, K>(d, c, l, Wh, Wh + H * K);  // TMEM: 512 columns; barrier inside
    constexpr uint32_t kBBytes = static_cast<uint32_t>(Sm::b_bytes);
    const float* wsrc = d.wpack + static_cast<int64_t>(4 * l) * H * H;  // the update operand blocks of layer l
    // W_u block 0: packed by the last optimizer step (at least two kernels back, or a
    // previous graph) - fetched before the dependency wait, overlapping the walk
    if (tid == 0) {
        mbar_expect_tx(&gb[0], kBBytes);
        bulk_g2s(Bw, wsrc, kBBytes, &gb[0]);
    }
    MessageBody<H, K, true, kZ, kMsgChunk> b{d, kZ ? d.tanh_emb : d.t[l], d.mu[l], l, c.lt};
    walk_edges<H, K>(d, c, b, ft);

    // ---- update GEMM over this CTA's atoms
    const int a0 = d.part_lo[blockIdx.x * kPartsPerCta], a1 = d.part_lo[(blockIdx.x + 1) * kPartsPerCta];
    umma::fence_before();
    __syncthreads();  // the walk's mu rows written (global), its TMEM columns and stages free
    umma::fence_after();
    const uint32_t tbase = *c.tslot;  // (the A tile below overwrites the walk region, slot included)
    if (tid < 2 * kMsgGroups * kStages) {  // the walk's TMA / MMA barriers: retired before the memory is reused
        uint64_t* wb = reinterpret_cast<uint64_t*>(lamm_edge_smem + EdgeSmem<K, kMsgGroups, kMsgChunk>::stage_bytes);
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(wb + tid)) : "memory");
    }
    __syncthreads();
    float* Ahi = reinterpret_cast<float*>(lamm_edge_smem +
                                          ((1024u - (smem_u32(lamm_edge_smem) & 1023u)) & 1023u));
    float* Alo = Ahi + kGemmM * H;
    const int warp = tid >> 5, lane = tid & 31, quad = warp & 3, part = warp >> 2;
    const uint32_t idesc = umma::idesc_tf32(kGemmM, NC);
    int have = 0;                   // W_u block resident in Bw (tid 0's view)
    uint32_t wpar = 0;              // parity of the next weights-barrier completion (tid 0)
    bool wpend = true;              // a weights load not yet waited for (tid 0)
    uint32_t tpar = 0;              // per-tile parity of the two MMA barriers
    for (int r0 = a0; r0 < a1; r0 += kGemmM) {
        const int nrows = min(kGemmM, a1 - r0);
        // A: mu rows [r0, r0 + nrows) into the SW128 K-major tile (16 KB per 32-column block)
#pragma unroll
        for (int it = 0; it < kGemmM * H / 4 / (kMsgGroups * H); ++it) {
            const int f = tid + kMsgGroups * H * it, row = f >> 5, c4 = f & 31;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < nrows) x = *reinterpret_cast<const float4*>(d.mu[l] + static_cast<int64_t>(r0 + row) * H + 4 * c4);
            const int off = (c4 >> 3) * kGemmM * 32 + row * 32 + (((c4 & 7) ^ (row & 7)) << 2);
            *reinterpret_cast<float4*>(Ahi + off) = x;
            *reinterpret_cast<float4*>(Alo + off) = make_float4(umma::tf32_trunc_lo(x.x), umma::tf32_trunc_lo(x.y),
                                                                umma::tf32_trunc_lo(x.z), umma::tf32_trunc_lo(x.w));
        }
        umma::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            for (int np = 0; np < 2; ++np) {
                if (have != np) {
                    // the block in Bw was read by the previous MMA group: wait for it, then reload
                    mbar_wait(&gb[1 + have], np == 1 ? tpar : tpar ^ 1u);
                    mbar_expect_tx(&gb[0], kBBytes);
                    bulk_g2s(Bw, wsrc + static_cast<int64_t>(np) * 2 * NC * H, kBBytes, &gb[0]);
                    have = np;
                    wpend = true;
                }
                if (wpend) {
                    mbar_wait(&gb[0], wpar);
                    wpar ^= 1u;
                    wpend = false;
                }
                umma::fence_after();
                const float* Blo = Bw + NC * H;
#pragma unroll
                for (int s = 0; s < H / 8; ++s)
                    umma::mma3(tbase + np * NC, umma::sw128_kdesc(Ahi, s, kGemmM), umma::sw128_kdesc(Alo, s, kGemmM),
                               umma::kdesc(Bw, s, H), umma::kdesc(Blo, s, H), idesc, s ? 1u : 0u);
                umma::commit(&gb[1 + np]);
            }
        }
        // epilogue per column block as its MMAs land: residual h_l (layer 0: E[Z]) + D
        const int row = quad * 32 + lane, atom = r0 + row;
        const bool live = row < nrows;
#pragma unroll
        for (int np = 0; np < 2; ++np) {
            const int c0 = np * NC + part * 16;
            float pre[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) pre[q] = 0.f;
            if (live) {
                const float* p = kZ ? d.emb + static_cast<int64_t>(__ldg(d.Z + atom) - 1) * H
                                    : d.h[l] + static_cast<int64_t>(atom) * H;
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    const float4 x = __ldg(reinterpret_cast<const float4*>(p + c0 + q));
                    pre[q] = x.x, pre[q + 1] = x.y, pre[q + 2] = x.z, pre[q + 3] = x.w;
                }
            }
            mbar_wait(&gb[1 + np], tpar);
            umma::fence_after();
            float v[16];
            umma::ld16(tbase + (static_cast<uint32_t>(quad * 32) << 16) + np * NC + part * 16, v);
            if (live) {
                float* ho = d.h[l + 1] + static_cast<int64_t>(atom) * H + c0;
                float* to = d.t[l + 1] + static_cast<int64_t>(atom) * H + c0;
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    const float h0 = pre[q] + v[q], h1 = pre[q + 1] + v[q + 1], h2 = pre[q + 2] + v[q + 2],
                                h3 = pre[q + 3] + v[q + 3];
                    *reinterpret_cast<float4*>(ho + q) = make_float4(h0, h1, h2, h3);
                    *reinterpret_cast<float4*>(to + q) = make_float4(tanhf(h0), tanhf(h1), tanhf(h2), tanhf(h3));
                }
            }
        }
        tpar ^= 1u;
        umma::fence_before();
        __syncthreads();  // the tile's MMAs and TMEM reads done before A / TMEM are reused
        umma::fence_after();
    }
    if (tid == 0 && wpend) mbar_wait(&gb[0], wpar);  // no tile: the prefetch still lands before exit
    umma::fence_before();
    __syncthreads();
    if (tid < 32) umma::tmem_dealloc(tbase, 512);
}

// Backward of the update GEMM fused with its weight gradient (H = 128):
//   gm = (gh W_u) (.) (1 - mu^2)        MMA1: A = the gh tile (shared, K-major canonical),
//                                       B = W_u block (K-major, TMA)       (S/model.cpp:380-390)
//   dW_u[:, cols] += gh^T mu[:, cols]   MMA2: A = gh^T from TMEM (lane = row b of W_u,
//                                       column = atom), B = the mu tile, MN-major
//                                       (128B_BASE32B) in the weights' place once MMA1
//                                       is done                            (S/model.cpp:381-383)
// Every shared-memory tile is written in its storage order (thread -> 16-byte
// chunk), so the staging stores are free of bank conflicts. The dW_u
// accumulator stays in TMEM across the CTA's tiles; one [H][NC] partial per CTA
// (its column block never changes: gridDim.x % NS == 0), summed by
// k_grad_reduce. TMEM: [0, NC) gm accumulator, [NC, 2 NC) dW_u, [256, 384)
// gh^T hi, [384, 512) gh^T lo.
template <int H>
struct BwdGemmSmem {
    static constexpr int NC = NodeGemmCfg<H>::NC;
    static constexpr size_t a_floats = 2 * kGemmM * H;  // gh tile hi | lo (MMA1's A)
    static constexpr size_t b_floats = NodeGemmCfg<H>::b_floats > 2 * kGemmM * NC ? NodeGemmCfg<H>::b_floats
                                                                                   : 2 * kGemmM * NC;
    static constexpr size_t bytes = 4 * (a_floats + b_floats) + 64 + 1024;  // + barriers, alignment slack
};

template <int H>
__global__ void __launch_bounds__(512, 1) k_bwd_gemm(Dev d, int l, const __grid_constant__ CUtensorMap ghmap) {
    using Cfg = NodeGemmCfg<H>;
    constexpr int NT = 512, NP4 = NT / 128;  // threads; column parts per TMEM lane quarter
    constexpr int NS = Cfg::NS, NC = Cfg::NC, CW = NC / NP4, Q = H / 4;
    static_assert(H == 128 && CW % 16 == 0, "fused update backward: H = 128");
    constexpr int MA = NC / 32;  // MN atoms of the mu tile
    extern __shared__ __align__(1024) unsigned char bwd_gemm_smem[];
    float* sm = reinterpret_cast<float*>(bwd_gemm_smem + ((1024u - (smem_u32(bwd_gemm_smem) & 1023u)) & 1023u));
    float* Ahi = sm;
    float* Alo = Ahi + kGemmM * H;
    float* Bhi = Alo + kGemmM * H;  // weights [NC][H] hi | lo, then the mu tile hi | lo
    uint64_t* bar = reinterpret_cast<uint64_t*>(Bhi + BwdGemmSmem<H>::b_floats);  // weights, MMA1, MMA2, gh TMA
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quad = warp & 3, part = warp >> 2;
    if (warp == 0) umma::tmem_alloc(tslot, 512);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], 1);
        mbar_init(&bar[3], 1);
        mbar_fence_init();
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = *tslot;
    const uint32_t tD1 = tbase, tD2 = tbase + NC, tAh = tbase + 256, tAl = tbase + 384;
    uint32_t gphase = 0;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t idesc = umma::idesc_tf32(kGemmM, NC);
    const uint32_t idesc_mn = umma::idesc_tf32(kGemmM, NC) | (1u << 16);  // B MN-major
    const int N = d.hdr->N;  // staged upload
    const int ntiles = (N + kGemmM - 1) / kGemmM * NS;
    const int np = blockIdx.x % NS;
    uint32_t wphase = 0, mphase = 0, dphase = 0;
    auto fetch_weights = [&]() {
        if (tid == 0) {
            const float* wsrc = d.wpack + static_cast<int64_t>(4 * l + 2) * H * H + static_cast<int64_t>(np) * 2 * NC * H;
            mbar_expect_tx(&bar[0], static_cast<uint32_t>(Cfg::b_floats * 4));
            bulk_g2s(Bhi, wsrc, static_cast<uint32_t>(Cfg::b_floats * 4), &bar[0]);
        }
    };
    if (static_cast<int>(blockIdx.x) < ntiles) fetch_weights();
    pdl_enter();
    const float* __restrict__ mu = d.mu[l];
    int done = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++done) {
        const int base = (tile / NS) * kGemmM;
        const int row = quad * 32 + lane, atom = base + row;
        const bool live = atom < N;
        const int c0 = np * NC + part * CW;
        if (done > 0) {  // MMA2 of the previous tile read TMEM A and the mu tile in B
            mbar_wait(&bar[2], dphase);
            dphase ^= 1u;
            umma::fence_after();
            fetch_weights();
        }
        // the gh tile by TMA (SWIZZLE_128B; raw fp32 = MMA1's tf32 hi operand), and this
        // thread's mu row segment for the epilogue
        if (tid == 0) {
            mbar_expect_tx(&bar[3], static_cast<uint32_t>(kGemmM * H * 4));
#pragma unroll
            for (int kb = 0; kb < H / 32; ++kb) umma::tma_load_2d(Ahi + kb * kGemmM * 32, &ghmap, kb * 32, base, &bar[3]);
        }
        float pre[CW];
#pragma unroll
        for (int q = 0; q < CW; q += 4) {
            const float4 x = live ? __ldg(reinterpret_cast<const float4*>(mu + static_cast<int64_t>(atom) * H + c0 + q))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            pre[q] = x.x, pre[q + 1] = x.y, pre[q + 2] = x.z, pre[q + 3] = x.w;
        }
        mbar_wait(&bar[3], gphase);
        gphase ^= 1u;
        {  // MMA1's lo operand: x - trunc_tf32(x) at the same swizzled positions
            constexpr int IT = kGemmM * Q / NT;
#pragma unroll
            for (int it = 0; it < IT; ++it) {
                const int c = tid + NT * it;
                const float4 x = *reinterpret_cast<const float4*>(Ahi + 4 * c);
                *reinterpret_cast<float4*>(Alo + 4 * c) =
                    make_float4(umma::tf32_trunc_lo(x.x), umma::tf32_trunc_lo(x.y), umma::tf32_trunc_lo(x.z),
                                umma::tf32_trunc_lo(x.w));
            }
        }
        // gh^T into TMEM from the staged tile: lane = channel b = row, columns = atoms
        // [part*32, part*32+32); element (atom m, channel b) of the SW128 tile sits in
        // K block b/32, row m, 16-byte chunk ((b%32)/4) ^ (m%8) (a warp reads one 128 B row)
        {
            const float* blk = Ahi + (row >> 5) * kGemmM * 32;
            const int j = (row & 31) >> 2, w = row & 3;
#pragma unroll
            for (int cc = 0; cc < kGemmM / NP4; cc += 16) {
                const int a0 = part * (kGemmM / NP4) + cc;
                float hv[16], lv[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const int m = a0 + q;
                    const float x = blk[m * 32 + ((j ^ (m & 7)) << 2) + w];  // rows past N: never read (MMA2 masks)
                    umma::split_tf32(base + m < N ? x : 0.f, hv[q], lv[q]);
                }
                umma::st16(tAh + lane_off + a0, hv);
                umma::st16(tAl + lane_off + a0, lv);
            }
        }
        umma::st_wait();
        umma::fence_proxy_async();
        umma::fence_before();
        __syncthreads();
        if (tid == 0) {
            mbar_wait(&bar[0], wphase);
            umma::fence_after();
            const float* Blo = Bhi + NC * H;
#pragma unroll
            for (int s = 0; s < H / 8; ++s)
                umma::mma3(tD1, umma::sw128_kdesc(Ahi, s, kGemmM), umma::sw128_kdesc(Alo, s, kGemmM),
                           umma::kdesc(Bhi, s, H), umma::kdesc(Blo, s, H), idesc, s ? 1u : 0u);
            umma::commit(&bar[1]);
        }
        wphase ^= 1u;
        // the mu tile for MMA2's B (N = this CTA's NC columns, K = atoms), MN-major
        // 128B_BASE32B, written chunk by chunk in storage order once MMA1 is done
        constexpr int MIT = kGemmM * NC / 4 / NT;
        float4 vm[MIT];
        int mo[MIT];
#pragma unroll
        for (int it = 0; it < MIT; ++it) {
            const int c = tid + NT * it;  // 16-byte chunk c of the tile in storage order
            const int mna = (c >> 5) % MA, kg = (c >> 5) / MA, kr = (c >> 3) & 3, x = (c >> 1) & 3, hl = c & 1;
            const int mn = mna * 32 + ((x ^ kr) << 3) + (hl << 2), k = kg * 4 + kr;  // column, atom
            vm[it] = base + k < N ? __ldg(reinterpret_cast<const float4*>(mu + static_cast<int64_t>(base + k) * H +
                                                                          np * NC + mn))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            mo[it] = 4 * c;
        }
        mbar_wait(&bar[1], mphase);
        mphase ^= 1u;
        umma::fence_after();
        {
            float* Mhi = Bhi;  // the weight block is free
            float* Mlo = Bhi + kGemmM * NC;
#pragma unroll
            for (int it = 0; it < MIT; ++it) {
                float4 h4, l4;
                umma::split_tf32(vm[it].x, h4.x, l4.x);
                umma::split_tf32(vm[it].y, h4.y, l4.y);
                umma::split_tf32(vm[it].z, h4.z, l4.z);
                umma::split_tf32(vm[it].w, h4.w, l4.w);
                *reinterpret_cast<float4*>(Mhi + mo[it]) = h4;
                *reinterpret_cast<float4*>(Mlo + mo[it]) = l4;
            }
            umma::fence_proxy_async();
            umma::fence_before();
            __syncthreads();
            if (tid == 0) {
                umma::fence_after();
#pragma unroll
                for (int s = 0; s < kGemmM / 8; ++s) {  // K-step s: atoms 8s..8s+7 = two 4-row groups
                    const uint64_t bh = umma::mn32_desc(Mhi + s * 2 * (MA << 7), MA);
                    const uint64_t bl = umma::mn32_desc(Mlo + s * 2 * (MA << 7), MA);
                    umma::mma_tf32_ts(tD2, tAh + s * 8, bh, idesc_mn, (done | s) ? 1u : 0u);
                    umma::mma_tf32_ts(tD2, tAh + s * 8, bl, idesc_mn, 1u);
                    umma::mma_tf32_ts(tD2, tAl + s * 8, bh, idesc_mn, 1u);
                }
                umma::commit(&bar[2]);
            }
        }
        // gm = (gh W_u) (.) (1 - mu^2)
#pragma unroll
        for (int cc = 0; cc < CW; cc += 16) {
            float v[16];
            umma::ld16(tD1 + lane_off + part * CW + cc, v);
            if (!live) continue;
            float* go = d.gm + static_cast<int64_t>(atom) * H + c0 + cc;
#pragma unroll
            for (int q = 0; q < 16; q += 4)
                *reinterpret_cast<float4*>(go + q) =
                    make_float4(v[q] * (1.f - pre[cc + q] * pre[cc + q]), v[q + 1] * (1.f - pre[cc + q + 1] * pre[cc + q + 1]),
                                v[q + 2] * (1.f - pre[cc + q + 2] * pre[cc + q + 2]),
                                v[q + 3] * (1.f - pre[cc + q + 3] * pre[cc + q + 3]));
        }
        umma::fence_before();
        __syncthreads();  // the gm accumulator and the A tile are drained before the next tile
        umma::fence_after();
    }
    // this CTA's dW_u partial: rows b = TMEM lanes, columns of block np
    if (done > 0) {
        mbar_wait(&bar[2], dphase);
        umma::fence_after();
    }
    const int row = quad * 32 + lane;
    float* pout = d.part_wu[l] + static_cast<int64_t>(blockIdx.x) * H * NC;
    if (done > 0)  // CTAs without a tile write nothing (k_grad_reduce reads CTAs < ntiles only)
#pragma unroll
        for (int cc = 0; cc < CW; cc += 16) {
            float v[16];
            umma::ld16(tD2 + lane_off + part * CW + cc, v);
#pragma unroll
            for (int k = 0; k < 16; k += 4)
                *reinterpret_cast<float4*>(pout + row * NC + part * CW + cc + k) =
                    make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
        }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tbase, 512);
}

template <int H>
struct DwuSmem {
    static constexpr size_t stage_floats = 4 * kGemmM * kGemmKC;  // A hi|lo, B hi|lo
    static constexpr size_t bytes = 4 * 2 * stage_floats + 64;
};

// dW_u[b][a] = sum_atoms gh[atom][b] mu[atom][a]: M = b (rows >= H zero), N = H,
// K = atoms in 32-atom chunks (double buffered); CTA c reduces a contiguous
// chunk range into one TMEM accumulator and writes one [H][H] partial.
// Staging: thread -> (column b, 4 consecutive atoms), coalesced scalar loads
// across the warp, one 16-byte store per operand into the canonical tile.
template <int H>
__global__ void __launch_bounds__(256, 1) k_dwu(Dev d, int l) {
    constexpr int TPC = 256 / H;                   // threads per column
    constexpr int GPT = (kGemmKC / 4) / TPC;       // 4-atom groups per thread
    constexpr uint32_t kCols = H < 32 ? 32 : H;
    float* sm = dyn_smem<float>();
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * DwuSmem<H>::stage_floats);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quad = warp & 3, half = warp >> 2;
    if (warp == 0) umma::tmem_alloc(tslot, kCols);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    for (int e = tid; e < 2 * DwuSmem<H>::stage_floats; e += blockDim.x) sm[e] = 0.f;  // rows >= H stay 0
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    pdl_enter();
    const uint32_t tbase = *tslot;
    const uint32_t idesc = umma::idesc_tf32(kGemmM, H);
    const int N = d.hdr->N;
    const int nch = (N + kGemmKC - 1) / kGemmKC;
    const int c0 = static_cast<int>((static_cast<int64_t>(nch) * blockIdx.x) / gridDim.x);
    const int c1 = static_cast<int>((static_cast<int64_t>(nch) * (blockIdx.x + 1)) / gridDim.x);
    const float* __restrict__ gh = d.gh;
    const float* __restrict__ mu = d.mu[l];
    const int col = tid % H, g0 = tid / H;
    int q = 0;
    for (int ch = c0; ch < c1; ++ch, ++q) {
        const int st = q & 1;
        if (q >= 2) mbar_wait(&bar[st], ((q - 2) >> 1) & 1);
        float* Ahi = sm + st * DwuSmem<H>::stage_floats;
        float* Alo = Ahi + kGemmM * kGemmKC;
        float* Bhi = Alo + kGemmM * kGemmKC;
        float* Blo = Bhi + kGemmM * kGemmKC;
        float gv[GPT][4], mv[GPT][4];
#pragma unroll
        for (int gi = 0; gi < GPT; ++gi)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int atom = ch * kGemmKC + 4 * (g0 + TPC * gi) + r;
                const bool ok = atom < N;
                gv[gi][r] = ok ? __ldg(gh + static_cast<int64_t>(atom) * H + col) : 0.f;
                mv[gi][r] = ok ? __ldg(mu + static_cast<int64_t>(atom) * H + col) : 0.f;
            }
#pragma unroll
        for (int gi = 0; gi < GPT; ++gi) {
            const int o = umma::kidx(col, 4 * (g0 + TPC * gi), kGemmKC);
            float4 h4, l4, hm, lm;
            umma::split_tf32(gv[gi][0], h4.x, l4.x);
            umma::split_tf32(gv[gi][1], h4.y, l4.y);
            umma::split_tf32(gv[gi][2], h4.z, l4.z);
            umma::split_tf32(gv[gi][3], h4.w, l4.w);
            umma::split_tf32(mv[gi][0], hm.x, lm.x);
            umma::split_tf32(mv[gi][1], hm.y, lm.y);
            umma::split_tf32(mv[gi][2], hm.z, lm.z);
            umma::split_tf32(mv[gi][3], hm.w, lm.w);
            *reinterpret_cast<float4*>(Ahi + o) = h4;
            *reinterpret_cast<float4*>(Alo + o) = l4;
            *reinterpret_cast<float4*>(Bhi + o) = hm;
            *reinterpret_cast<float4*>(Blo + o) = lm;
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
    const int row = quad * 32 + lane;
    constexpr int CW = H / 2;
    float* part = d.part_wu[l] + static_cast<int64_t>(blockIdx.x) * H * H;
#pragma unroll
    for (int c = 0; c < CW; c += 16) {
        float v[16];
        umma::ld16(tbase + (static_cast<uint32_t>(quad * 32) << 16) + half * CW + c, v);
        if (row < H)
#pragma unroll
            for (int k = 0; k < 16; k += 4)
                *reinterpret_cast<float4*>(part + row * H + half * CW + c + k) =
                    q > 0 ? make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tbase, kCols);
}

}  // namespace lamm_b200
