// edge_kernels.cuh - the four message-passing kernels of the step (forward
// message, force head, head backward, layer backward), sm_100a.
//
// Shape of every kernel: the CSR edge list (grouped by destination atom i, j
// ascending) is cut by k_nbr_fill into Q = gridDim.x * 12 cost-balanced (edges + 4 per atom)
// partitions of whole atoms. A CTA runs kGroups independent "groups" of H
// threads; thread a of a group owns feature channel a. A group walks its
// partition's edges in order:
//   * edge metadata (j, i, unit/fcut, fcut*rbf) arrives in shared memory in
//     64-edge chunks by TMA bulk copies (cp.async.bulk + mbarrier, double
//     buffered);
//   * edges are consumed in blocks of 8 (16 in the message walk): vector reads of
//     j/i, one coalesced source-row gather per edge and thread, the next block's
//     issued before the current one is consumed (the CSR is padded
//     so every staged j is a valid atom), a uniform validity mask, and the
//     per-destination segmented sum as a register accumulation flushed when the
//     destination changes;
//   * for H = 128 the per-edge radial filter W_f (fcut rbf_e) of the message and
//     of the layer backward runs on the tensor core: the group leader issues
//     D[a][e] = sum_k W_f[a][k] fcut rbf[e][k] (M = 128 channels = TMEM lanes,
//     N = 64 edges, K = 16, 3xTF32 tcgen05.mma) for chunk c+1 while the group
//     drains chunk c, and thread a reads its filter row a block at a time with
//     tcgen05.ld 32x32b.x8 / .x16.
// The message walk of the train step is followed, in the same kernel, by the
// update GEMM of the CTA's own atoms (k_message_update, gemm_kernels.cuh).
// No atomics: parameter-gradient contributions accumulate in thread-owned
// registers / shared memory and leave each kernel as one per-CTA partial,
// summed across CTAs in index order by k_grad_reduce.
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"
#include "umma.cuh"

namespace lamm_b200 {

constexpr int kGroups = 4;   // independent edge streams per CTA (default geometry)
constexpr int kChunk = 64;   // edges per staged chunk (= MMA N of the filter)
constexpr int kStages = 2;   // staging double buffer
// k_nbr_fill cuts kPartsPerCta partitions per CTA; a kernel with G groups gives
// each group kPartsPerCta / G consecutive ones (G in {2, 3, 4, 6})
constexpr int kPartsPerCta = 12;
// geometry of the message kernel (measured: 6 groups of 32-edge chunks, 24
// warps per SM, is slower than 4 x 64 - the per-chunk overhead doubles)
constexpr int kMsgGroups = 4;
constexpr int kMsgChunk = 64;
// the force edges need no TMEM and fit 6 groups (768 threads, <= 85 registers)
constexpr int kForceGroups = 6;

// fcut*rbf of the edges for the tensor core: K-major canonical ("interleaved")
// layout in blocks of 8 edges, element (e, k) at ((e/8)*(K/4) + k/4)*32 +
// (e%8)*4 + k%4, as a tf32 hi part and an fp32 lo remainder (hi + lo == fcut*rbf).
template <int K>
__host__ __device__ __forceinline__ int64_t rbf_idx(int64_t e, int k) {
    return (((e >> 3) * (K / 4) + (k >> 2)) << 5) + ((e & 7) << 2) + (k & 3);
}

template <int K, int C = kChunk>
struct EdgeStage {
    static constexpr int kC = C;
    int32_t col[C];
    int32_t dst[C];
    uint32_t segw[8];  // segment-start bits of the 256 edges from word (cb >> 5) & ~3
    float4 geo[C];     // u_x, u_y, u_z, fcut
    float fcp[C * K];  // fcut*rbf, edge-major
    float fch[C * K];  // fcut*rbf, canonical tf32 hi (tensor-core filter)
    float fcl[C * K];  // fcut*rbf, canonical lo
    float2 sij[C];     // train-step head backward: s_ij and gF_i.u_ij (k_loss)
    int32_t colz[C];   // Z_j - 1 (layer-0 layer backward)
};

// --------------------------------------------------------------- PTX glue --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Packed fp32 pair FMA (FFMA2 on sm_100a): two IEEE fmaf in one instruction.
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t f32x2_splat(float x) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void f32x2_unpack(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ void group_sync(int g, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(nthreads) : "memory");
}

enum StageParts : int { kPartGeo = 1, kPartPlain = 2, kPartCanon = 4, kPartSij = 8, kPartColZ = 16, kPartZRow = 32 };

// One TMA stage: edges [cb, cb + n), n = min(kChunk, e1 - cb) rounded up to a
// whole 8-edge block (the tail reads into the CSR padding).
template <int K, int C, int kB = 8>
__device__ __forceinline__ void stage_chunk(const Dev& d, EdgeStage<K, C>& s, uint64_t* b, int cb, int e1, int parts) {
    const int n = min(C, ((e1 - cb) + kB - 1) & ~(kB - 1));
    uint32_t bytes = 8u * n + 32u;
    if (parts & kPartGeo) bytes += 16u * n;
    if (parts & kPartPlain) bytes += 4u * K * n;
    if (parts & kPartCanon) bytes += 8u * K * n;
    if (parts & kPartSij) bytes += 8u * n;
    if (parts & kPartZRow) bytes += 4u * n;
    mbar_expect_tx(b, bytes);
    bulk_g2s(s.col, ((parts & kPartColZ) ? d.colz : d.col) + cb, 4 * n, b);  // kPartColZ: source rows Z_j - 1
    bulk_g2s(s.dst, d.dst + cb, 4 * n, b);
    bulk_g2s(s.segw, d.segw + ((cb >> 5) & ~3), 32, b);
    if (parts & kPartGeo) bulk_g2s(s.geo, d.geo + cb, 16 * n, b);
    if (parts & kPartPlain) bulk_g2s(s.fcp, d.rbfp + static_cast<int64_t>(cb) * K, 4 * K * n, b);
    if (parts & kPartCanon) {
        bulk_g2s(s.fch, d.rbf + static_cast<int64_t>(cb) * K, 4 * K * n, b);
        bulk_g2s(s.fcl, d.rbfl + static_cast<int64_t>(cb) * K, 4 * K * n, b);
    }
    if (parts & kPartSij) bulk_g2s(s.sij, d.sij + cb, 8u * n, b);
    if (parts & kPartZRow) bulk_g2s(s.colz, d.colz + cb, 4u * n, b);
}

// Shared-memory layout common to the edge kernels: per group kStages staged
// chunks + TMA barriers + filter-MMA barriers, then the kernel's own region.
template <int K, int G = kGroups, int C = kChunk>
struct EdgeSmem {
    static constexpr size_t stage_bytes = sizeof(EdgeStage<K, C>) * kStages * G;
    static constexpr size_t bar_bytes = 16 * kStages * G * 2 + 16;
    static constexpr size_t extra_offset = stage_bytes + bar_bytes;
};

template <int H, int K, int G = kGroups, int C = kChunk>
struct EdgeCta {
    static constexpr int kG = G, kC = C;
    EdgeStage<K, C>* st;
    uint64_t* bar;   // [kStages] TMA
    uint64_t* mbar;  // [kStages] filter MMA
    uint32_t* tslot;
    char* extra;
    int g, lt, q, lo, hi;
    bool late;
};

// late_parts: the partitions were cut by the previous kernel (k_nbr_fill before
// the layer-0 message), so they are read after the dependency wait; otherwise
// they are at least two kernels old and load with the prologue.
template <int H, int K, int G = kGroups, int C = kChunk>
__device__ __forceinline__ EdgeCta<H, K, G, C> edge_prologue(const Dev& d, bool late_parts = false) {
    static_assert(kPartsPerCta % G == 0, "groups must divide the partitions of a CTA");
    extern __shared__ __align__(128) unsigned char lamm_edge_smem[];
    using Smem = EdgeSmem<K, G, C>;
    EdgeCta<H, K, G, C> c;
    c.g = threadIdx.x / H;
    c.lt = threadIdx.x % H;
    c.st = reinterpret_cast<EdgeStage<K, C>*>(lamm_edge_smem) + c.g * kStages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(lamm_edge_smem + Smem::stage_bytes);
    c.bar = bars + c.g * kStages;
    c.mbar = bars + G * kStages + c.g * kStages;
    c.tslot = reinterpret_cast<uint32_t*>(bars + 2 * G * kStages);
    c.extra = reinterpret_cast<char*>(lamm_edge_smem + Smem::extra_offset);
    if (c.lt == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&c.bar[s], 1), mbar_init(&c.mbar[s], 1);
        mbar_fence_init();
    }
    c.q = blockIdx.x * kPartsPerCta + c.g * (kPartsPerCta / G);
    c.late = late_parts;
    c.lo = c.hi = 0;
    if (!late_parts) c.lo = d.part_lo[c.q], c.hi = d.part_lo[c.q + kPartsPerCta / G];
    return c;
}

// Tensor-core filter state of a group: W_f as canonical hi/lo K-major tiles in
// shared memory, this group's 2 x 64 TMEM columns.
struct FilterTc {
    const float* Wh;
    const float* Wl;
    uint32_t tg;  // TMEM address of the group's first column
    uint32_t idesc;
};

template <int K, int C>
__device__ __forceinline__ void filter_mma(uint32_t tcol, const FilterTc& f, const EdgeStage<K, C>& s) {
    umma::fence_after();
#pragma unroll
    for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t ah = umma::kdesc(f.Wh, ks, K), al = umma::kdesc(f.Wl, ks, K);
        const uint64_t bh = umma::sdesc(s.fch + ks * 64, 128u, (K / 4) * 128u);
        const uint64_t bl = umma::sdesc(s.fcl + ks * 64, 128u, (K / 4) * 128u);
        umma::mma3(tcol, ah, al, bh, bl, f.idesc, ks ? 1u : 0u);
    }
}

// Walks the edges of the group's atoms [lo, hi). Body provides:
//   static constexpr bool kFilter;   tensor-core filter values passed to edge()
//   static constexpr int  kParts;    staged arrays besides col/dst
//   struct Reg;  void load(const EdgeStage<K>&, int e, int j, Reg&);
//   void edge(const EdgeStage<K>&, int e, const Reg&, float filter, unsigned on);
//        (on is 1 for the edges of the current segment, 0 otherwise: bodies
//        predicate their accumulation on it; every edge is "on" exactly once)
//   void begin(int i); void end(int i);     destination-atom brackets
//   static constexpr bool kPrepare;  if set, prepare(st, e0) runs once per 8-edge
//        block before its segments, warp-converged (per-edge scalar work done by 8
//        lanes and broadcast with shuffles instead of by every channel thread)
//   static constexpr bool kBlockHook;  if set, block(st, e0, r, ulo, uhi) runs once
//        per 8-edge block after its segments (segment-independent per-edge work;
//        edges [ulo, uhi) of the block are valid); group-uniform, may group_sync
template <int H, int K, int G, int C, class Body>
__device__ __forceinline__ void walk_edges(const Dev& d, const EdgeCta<H, K, G, C>& c, Body& body, const FilterTc& ft) {
    constexpr bool kF = Body::kFilter;
    constexpr int parts = Body::kParts | (kF ? kPartCanon : 0);
    // The CSR (partitions, row_ptr, edge metadata) and the weights are at least two
    // kernels old unless c.late (layer-0 message): the first two chunks are staged
    // and the first filter MMA issued before the dependency wait, overlapping the
    // previous kernel's tail; the source-row gathers and body.begin come after it.
    if (c.late) pdl_enter();
    int plo = c.lo, phi = c.hi;
    if (c.late) plo = d.part_lo[c.q], phi = d.part_lo[c.q + kPartsPerCta / G];
    if (plo >= phi) {
        if (!c.late) pdl_enter();
        return;
    }
    const int e0 = d.row_ptr[plo], e1 = d.row_ptr[phi];
    // the staging / MMA-issuing thread: lane 0 of warp g % (H/32) of the group, so the
    // four groups' leaders sit on different SM sub-partitions (warp id % 4)
    const bool lead = c.lt == 32 * (c.g % (H / 32));
    const uint32_t quad = (threadIdx.x >> 5) & 3;
    constexpr int kB = Body::kBlock;  // edges per block (8 or 16)
    constexpr unsigned kFull = (1u << kB) - 1u;
    const int base = e0 & ~(kB - 1);  // chunks start on whole blocks
    const int nchunks = (e1 - base + C - 1) / C;
    if (lead && e1 > e0) {
        stage_chunk<K, C, kB>(d, c.st[0], &c.bar[0], base, e1, parts);
        if (nchunks > 1) stage_chunk<K, C, kB>(d, c.st[1], &c.bar[1], base + C, e1, parts);
        if constexpr (kF) {
            mbar_wait(&c.bar[0], 0);
            filter_mma<K, C>(ft.tg, ft, c.st[0]);
            umma::commit(&c.mbar[0]);
        }
    }
    if (!c.late) pdl_enter();
    int cur = plo;
    body.begin(cur);
    if (e1 > e0) {
        // gathers of the next block are issued before the current block is
        // consumed, across chunk boundaries (the next chunk's stage is waited for
        // at the start of the current chunk)
        typename Body::Reg rn[kB];
        auto load_block = [&](const EdgeStage<K, C>& sst, int blk) {
#pragma unroll
            for (int q = 0; q < kB / 4; ++q) {
                const int4 j4 = reinterpret_cast<const int4*>(sst.col)[(kB / 4) * blk + q];
                body.load(sst, blk * kB + 4 * q, j4.x, rn[4 * q]);
                body.load(sst, blk * kB + 4 * q + 1, j4.y, rn[4 * q + 1]);
                body.load(sst, blk * kB + 4 * q + 2, j4.z, rn[4 * q + 2]);
                body.load(sst, blk * kB + 4 * q + 3, j4.w, rn[4 * q + 3]);
            }
        };
        mbar_wait(&c.bar[0], 0);
        load_block(c.st[0], (e0 - base) / kB);
        for (int k = 0; k < nchunks; ++k) {
            const int s = k & 1;
            const bool more = k + 1 < nchunks;
            if (more) {
                mbar_wait(&c.bar[s ^ 1], ((k + 1) >> 1) & 1);
                if constexpr (kF) {
                    if (lead) {  // next chunk's filter overlaps this chunk's drain
                        filter_mma<K, C>(ft.tg + (s ^ 1) * C, ft, c.st[s ^ 1]);
                        umma::commit(&c.mbar[s ^ 1]);
                    }
                }
            }
            if constexpr (kF) {
                mbar_wait(&c.mbar[s], (k >> 1) & 1);
                umma::fence_after();
            }
            const EdgeStage<K, C>& st = c.st[s];
            const int cb = base + k * C;
            const int ea = max(cb, e0) - cb, eb = min(cb + C, e1) - cb;
            const uint32_t trow = ft.tg + s * C + (quad * 32u << 16);
            const int blk0 = ea / kB, blk1 = (eb + kB - 1) / kB;
#pragma unroll(Body::kUnroll)
            for (int blk = blk0; blk < blk1; ++blk) {
                typename Body::Reg r[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u) r[u] = rn[u];
                if (blk + 1 < blk1) load_block(st, blk + 1);
                else if (more) load_block(c.st[s ^ 1], 0);  // first block of the next chunk
                const int ulo = max(ea - blk * kB, 0), uhi = min(eb - blk * kB, kB);
                if constexpr (Body::kPrepare) body.prepare(st, blk * kB);
                float f[kB];
                if constexpr (kF) {
                    if constexpr (kB == 16) umma::ld16(trow + blk * kB, f);
                    else umma::ld8(trow + blk * kB, f);
                } else {
#pragma unroll
                    for (int u = 0; u < kB; ++u) f[u] = 0.f;
                }
                // destination segments of the block: one flush call site per
                // block (keeps end()/begin() inlined once), branch-free edges
                const unsigned vm = ((1u << uhi) - 1u) & ~((1u << ulo) - 1u);
                const int bp = cb - (((cb >> 5) & ~3) << 5) + blk * kB;  // bit of the block's first edge
                unsigned seg = (((st.segw[bp >> 5] >> (bp & 31)) & kFull) | (1u << ulo)) & vm;
                if (seg == 1u && vm == kFull && st.dst[blk * kB] == cur) {
                    // the common block: all edges of the current destination (no
                    // segment start inside): the unpredicated body
#pragma unroll
                    for (int u = 0; u < kB; ++u) body.edge(st, blk * kB + u, r[u], f[u], 1u);
                    seg = 0u;
                }
                while (seg) {
                    const int u0 = __ffs(seg) - 1;
                    seg &= seg - 1u;
                    const int u1 = seg ? __ffs(seg) - 1 : uhi;
                    const int i = st.dst[blk * kB + u0];
                    if (i != cur) {
                        do {
                            body.end(cur);
                            ++cur;
                            body.begin(cur);
                        } while (cur < i);
                    }
                    const unsigned on = ((1u << u1) - 1u) & ~((1u << u0) - 1u);  // this segment's edges
#pragma unroll
                    for (int u = 0; u < kB; ++u) body.edge(st, blk * kB + u, r[u], f[u], (on >> u) & 1u);
                }
                if constexpr (Body::kBlockHook) body.block(st, blk * kB, r, ulo, uhi);
            }
            if constexpr (kF) umma::fence_before();
            group_sync(c.g, H);  // every thread is done with this stage (smem + TMEM)
            if (lead && k + 2 < nchunks) stage_chunk<K, C, kB>(d, c.st[s], &c.bar[s], base + (k + 2) * C, e1, parts);
        }
    }
    body.end(cur);
    for (int i = cur + 1; i < phi; ++i) {
        body.begin(i);
        body.end(i);
    }
}

// Loads W_f of layer l as canonical hi/lo tiles and allocates the CTA's TMEM
// (all 512 columns: kGroups x 2 stages x 64). Call from all threads.
template <int H, int K, int G, int C>
__device__ __forceinline__ FilterTc filter_setup(const Dev& d, const EdgeCta<H, K, G, C>& c, int l, float* Wh, float* Wl) {
    if (threadIdx.x < 32) umma::tmem_alloc(c.tslot, 512);
    const float* __restrict__ wf = d.wf[l];
    for (int idx = threadIdx.x; idx < H * K; idx += blockDim.x) {
        const int a = idx / K, k = idx % K;
        umma::split_tf32(wf[idx], Wh[umma::kidx(a, k, K)], Wl[umma::kidx(a, k, K)]);
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    static_assert(G * 2 * C <= 512, "TMEM: groups x 2 stages x chunk columns");
    return FilterTc{Wh, Wl, *c.tslot + static_cast<uint32_t>(c.g * 2 * C), umma::idesc_tf32(128, C)};
}

__device__ __forceinline__ void filter_teardown(const uint32_t* tslot) {
    umma::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_dealloc(*tslot, 512);
}

template <int K, int C>
__device__ __forceinline__ float filter_ffma(const float (&w)[K], const EdgeStage<K, C>& s, int e) {
    const float4* fr = reinterpret_cast<const float4*>(s.fcp + e * K);
    float f = 0.f;
#pragma unroll
    for (int k4 = 0; k4 < K / 4; ++k4) {
        const float4 q = fr[k4];
        f = fmaf(w[4 * k4], q.x, f);
        f = fmaf(w[4 * k4 + 1], q.y, f);
        f = fmaf(w[4 * k4 + 2], q.z, f);
        f = fmaf(w[4 * k4 + 3], q.w, f);
    }
    return f;
}

template <int H, int K>
struct EdgeKernelSmem {
    static constexpr bool TC = H == 128;
    static constexpr size_t base = EdgeSmem<K>::extra_offset;
    static constexpr size_t filter = TC ? 4 * 2 * H * K : 0;
    static constexpr size_t one_cta = 120 * 1024;  // > half the SM: one CTA owns the 512 TMEM columns
    static size_t pad(size_t b) { return TC && b < one_cta ? one_cta : b; }
    static size_t message() { return pad(EdgeSmem<K, kMsgGroups, kMsgChunk>::extra_offset + filter); }
    static size_t force(int) { return EdgeSmem<K, kForceGroups, kChunk>::extra_offset; }
    static size_t head(int D) { return base + 4 * kGroups * (3 * D * H + D * K); }
    static size_t bwd() { return pad(base + filter + 4 * kGroups * H * K); }
};

// ---------------------------------------------------------------- message --
// m_i[a] = sum_j t_j[a] * sum_k Wf[a,k] fcut_ij rbf_ijk ; mu_i = tanh(m_i)   (S/model.cpp:78-93)
// kZ: layer 0, whose source rows are tanh(E)[Z_j - 1] (compile-time, so layers
// >= 1 carry no predicated-off Z gathers)
template <int H, int K, bool TC, bool kZ, int C = kChunk>
struct MessageBody {
    static constexpr bool kFilter = TC;
    // layer 0 stages Z_j - 1 (k_nbr_fill) in place of j: no dependent Z load per edge
    static constexpr int kParts = (TC ? 0 : kPartPlain) | (kZ ? kPartColZ : 0);
    static constexpr bool kBlockHook = false;
    static constexpr bool kPrepare = false;
    static constexpr int kUnroll = 1;  // block loop unroll (2: the r/rn register roles alternate)
    static constexpr int kBlock = 16;  // edges per block of the walk
    struct Reg {
        float t;
    };
    const Dev& d;
    const float* __restrict__ tsrc;
    float* mu;
    int l, a;
    float w[K];
    float m;
    __device__ void load(const EdgeStage<K, C>&, int, int j, Reg& r) const {
        r.t = __ldg(tsrc + static_cast<int64_t>(j) * H + a);  // j = Z_j - 1 at layer 0 (kPartColZ)
    }
    __device__ void edge(const EdgeStage<K, C>& s, int e, const Reg& r, float f, unsigned on) {
        if constexpr (!TC) f = filter_ffma<K>(w, s, e);
        m = fmaf(r.t, on ? f : 0.f, m);
    }
    __device__ void begin(int) { m = 0.f; }
    __device__ void end(int i) { mu[static_cast<int64_t>(i) * H + a] = tanhf(m); }
};

template <int H, int K, bool kZ>
__global__ void __launch_bounds__(kMsgGroups* H, 1) k_edge_message(Dev d, int l) {
    constexpr bool TC = EdgeKernelSmem<H, K>::TC;
    EdgeCta<H, K, kMsgGroups, kMsgChunk> c = edge_prologue<H, K, kMsgGroups, kMsgChunk>(d, kZ);
    FilterTc ft{};
    if constexpr (TC) {
        float* Wh = reinterpret_cast<float*>(c.extra);
        ft = filter_setup<H, K>(d, c, l, Wh, Wh + H * K);
    } else {
        __syncthreads();
    }
    MessageBody<H, K, TC, kZ, kMsgChunk> b{d, kZ ? d.tanh_emb : d.t[l], d.mu[l], l, c.lt};
    if constexpr (!TC) {
#pragma unroll
        for (int k = 0; k < K; ++k) b.w[k] = d.wf[l][c.lt * K + k];
    }
    walk_edges<H, K>(d, c, b, ft);
    if constexpr (TC) filter_teardown(c.tslot);
}

// ------------------------------------------------------------ force head --
// F_i^d = sum_j w_ijd fcut_ij u_ij with w_ijd = A_i^d + A_j^d + sum_a Wb[a,d] T_ia T_ja
// + sum_k Wc[k,d] rbf_ijk and A = T Wa (S/model.cpp:223-253), re-associated per
// destination atom so that every edge costs one T_j gather and 3 FMAs:
//   Y_i[a] = sum_j T_ja fcut u_ij,  U_i = sum_j fcut u_ij,  V_i[k] = sum_j fcut rbf_ijk u_ij
//   F_i^d = sum_a [ Wa[a,d] (T_ia U_i + Y_i[a]) + Wb[a,d] T_ia Y_i[a] ] + sum_k Wc[k,d] V_i[k]
// (sum_j A_j^d fcut u_ij = sum_a Wa[a,d] Y_i[a]). k_edge_force walks the edges
// and writes the per-atom features Yf[i] = [Y (H x 3) | U (3) | V (K x 3)];
// k_force_out contracts them with the head weights, warp per atom.
template <int H, int K>
struct ForceBody {
    static constexpr bool kFilter = false;
    static constexpr int kParts = kPartGeo | kPartPlain;
    static constexpr bool kBlockHook = false;
    static constexpr bool kPrepare = false;
    static constexpr int kUnroll = 1;  // block loop unroll (2: the r/rn register roles alternate)
    static constexpr int kBlock = 8;  // edges per block of the walk
    static constexpr int kYW = (3 * H + 3 + 3 * K + 3) / 4 * 4;  // per-atom feature floats (16-byte rows)
    struct Reg {
        float t;
    };
    const Dev& d;
    const float* __restrict__ T;
    int a, L;
    bool kv;  // lanes 0..K-1 of warp g % (H/32): the channel-independent sums (one warp per
              // group, a different SM sub-partition per group)
    int k;
    uint64_t Y01;  // (Y0, Y1) as a packed fp32 pair: one FFMA2 per edge for x and y
    float Y2, U0, U1, U2, V0, V1, V2;
    __device__ void load(const EdgeStage<K>&, int, int j, Reg& r) const {
        r.t = __ldg(T + static_cast<int64_t>(j) * H + a);  // t[L], L >= 1 (ctx creation)
    }
    // branch-free: edges outside the segment contribute exact zeros
    __device__ void edge(const EdgeStage<K>& s, int e, const Reg& r, float, unsigned on) {
        const float4 gv = s.geo[e];
        const float mk = on ? 1.f : 0.f;
        const float fw = gv.w * mk;
        const float tf = r.t * fw;
        uint64_t gxy;
        asm("mov.b64 %0, {%1, %2};" : "=l"(gxy) : "f"(gv.x), "f"(gv.y));
        Y01 = ffma2(f32x2_splat(tf), gxy, Y01);
        Y2 = fmaf(tf, gv.z, Y2);
        if (kv) {  // channel-independent sums
            U0 = fmaf(fw, gv.x, U0);
            U1 = fmaf(fw, gv.y, U1);
            U2 = fmaf(fw, gv.z, U2);
            const float fr = s.fcp[e * K + k] * mk;
            V0 = fmaf(fr, gv.x, V0);
            V1 = fmaf(fr, gv.y, V1);
            V2 = fmaf(fr, gv.z, V2);
        }
    }
    __device__ void begin(int) {
        Y01 = 0ull;
        Y2 = U0 = U1 = U2 = V0 = V1 = V2 = 0.f;
    }
    __device__ void end(int i) {
        float* y = d.Yf + static_cast<int64_t>(i) * kYW;
        float Y0, Y1;
        f32x2_unpack(Y01, Y0, Y1);
        y[a] = Y0, y[H + a] = Y1, y[2 * H + a] = Y2;
        if (kv && k == 0) y[3 * H] = U0, y[3 * H + 1] = U1, y[3 * H + 2] = U2;
        if (kv) y[3 * H + 3 + k] = V0, y[3 * H + 3 + K + k] = V1, y[3 * H + 3 + 2 * K + k] = V2;
    }
};

template <int H, int K>
__global__ void __launch_bounds__(kForceGroups* H, 1) k_edge_force(Dev d) {
    EdgeCta<H, K, kForceGroups> c = edge_prologue<H, K, kForceGroups>(d);
    __syncthreads();
    const int kw = c.g % (H / 32);
    ForceBody<H, K> b{d, d.t[d.L], c.lt, d.L,
                      (c.lt >> 5) == kw && (c.lt & 31) < K, c.lt & 31};
    walk_edges<H, K>(d, c, b, FilterTc{});
}

// F_i[d][x] from the per-atom features, warp per atom: lane owns channels
// [lane*C, lane*C+C) and k = lane (< K); 3D partial sums per lane, one warp
// reduce-scatter (lane o ends with output o), coalesced store of F_i. The head
// weights sit transposed in shared memory ([D][H] rows, vector reads).
template <int H, int K, int R0>
__device__ __forceinline__ void force_out_round(const float* WaT, const float* WbT, const float* WcT, int D, int ND,
                                                int lane, const float (&ti)[H / 32], const float (&yv)[3][H / 32],
                                                const float (&u)[3], const float (&vk)[3], float* out) {
    constexpr int C = H / 32;
    float v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        const int idx = R0 + k, dd = idx / 3, x = idx % 3;
        float s = 0.f;
        if (idx < ND) {
            const VecF<C> wa = ldv<C>(WaT + dd * H + lane * C);
            const VecF<C> wb = ldv<C>(WbT + dd * H + lane * C);
#pragma unroll
            for (int cc = 0; cc < C; ++cc) {
                s = fmaf(wa.v[cc], fmaf(ti[cc], u[x], yv[x][cc]), s);
                s = fmaf(wb.v[cc], ti[cc] * yv[x][cc], s);
            }
            if (lane < K) s = fmaf(WcT[dd * 32 + lane], vk[x], s);
        }
        v[k] = s;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < o; ++k) {
            const float send = up ? v[k] : v[k + o];
            const float keep = up ? v[k + o] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    if (R0 + lane < ND) out[R0 + lane] = v[0];
}

// own_head: the train step reads only each atom's own head (its sample's
// dataset index) from F, so only those three components are formed.
template <int H, int K>
__global__ void __launch_bounds__(256) k_force_out(Dev d, int own_head) {
    constexpr int C = H / 32, YW = ForceBody<H, K>::kYW;
    __shared__ __align__(16) float WaT[kMaxHeads * H], WbT[kMaxHeads * H], WcT[kMaxHeads * 32], WeT[kMaxHeads * H];
    const int D = d.D, ND = 3 * D, L = d.L;
    for (int idx = threadIdx.x; idx < D * H; idx += blockDim.x) {
        const int dd = idx / H, aa = idx % H;
        WaT[idx] = d.wfh[aa * D + dd];
        WbT[idx] = d.wfh[(H + aa) * D + dd];
        WeT[idx] = d.we[aa * D + dd];
    }
    for (int idx = threadIdx.x; idx < D * 32; idx += blockDim.x) {
        const int dd = idx / 32, k = idx % 32;
        WcT[idx] = k < K ? d.wfh[(2 * H + k) * D + dd] : 0.f;
    }
    __syncthreads();
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const float* __restrict__ T = L > 0 ? d.t[L] : d.tanh_emb;
    const int N = d.hdr->N;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
        const float* y = d.Yf + static_cast<int64_t>(i) * YW;
        const int row = L > 0 ? i : __ldg(d.Z + i) - 1;
        float ti[C], yv[3][C];
        const VecF<C> tv = ldv<C>(T + static_cast<int64_t>(row) * H + lane * C);
        const VecF<C> y0 = ldv<C>(y + lane * C), y1 = ldv<C>(y + H + lane * C), y2 = ldv<C>(y + 2 * H + lane * C);
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
            ti[cc] = tv.v[cc];
            yv[0][cc] = y0.v[cc], yv[1][cc] = y1.v[cc], yv[2][cc] = y2.v[cc];
        }
        const float u[3] = {y[3 * H], y[3 * H + 1], y[3 * H + 2]};
        float vk[3] = {0.f, 0.f, 0.f};
        if (lane < K) vk[0] = y[3 * H + 3 + lane], vk[1] = y[3 * H + 3 + K + lane], vk[2] = y[3 * H + 3 + 2 * K + lane];
        float* out = d.F + static_cast<int64_t>(i) * ND;
        if (own_head) {
            const int dd = d.chan[i];
            const VecF<C> wa = ldv<C>(WaT + dd * H + lane * C);
            const VecF<C> wb = ldv<C>(WbT + dd * H + lane * C);
            const float wc = lane < K ? WcT[dd * 32 + lane] : 0.f;
            float sx[3];
#pragma unroll
            for (int x = 0; x < 3; ++x) {
                float acc = 0.f;
#pragma unroll
                for (int cc = 0; cc < C; ++cc) {
                    acc = fmaf(wa.v[cc], fmaf(ti[cc], u[x], yv[x][cc]), acc);
                    acc = fmaf(wb.v[cc], ti[cc] * yv[x][cc], acc);
                }
                sx[x] = fmaf(wc, vk[x], acc);
            }
#pragma unroll
            for (int x = 0; x < 3; ++x) sx[x] = warp_sum(sx[x]);
            if (lane < 3) out[dd * 3 + lane] = lane == 0 ? sx[0] : (lane == 1 ? sx[1] : sx[2]);
            // the atom's share of its sample's loss (k_loss sums them per sample):
            // energy e_i = sum_a h^L[i,a] W_e[a,d] (S/model.cpp:208-218) and the
            // Eq. (5) force term with its gradient (S/loss.cpp:186-212)
            const VecF<C> hv = ldv<C>(d.h[L] + static_cast<int64_t>(i) * H + lane * C);
            const VecF<C> we = ldv<C>(WeT + dd * H + lane * C);
            double e = 0.0;
#pragma unroll
            for (int cc = 0; cc < C; ++cc) e = fma(static_cast<double>(hv.v[cc]), static_cast<double>(we.v[cc]), e);
            e = warp_sum_d(e);
            if (lane == 0) {
                float4 gc = make_float4(0.f, 0.f, 0.f, 0.f);
                double ft = 0.0;
                const double ws = d.fw[i];  // 0 unless the sample trains forces
                if (ws != 0.0) {
                    double df[3], sq = 0.0;
#pragma unroll
                    for (int x = 0; x < 3; ++x) {
                        df[x] = static_cast<double>(sx[x]) - d.Fn[3 * static_cast<int64_t>(i) + x];
                        sq += df[x] * df[x];
                    }
                    const double dist = sqrt(sq);
                    ft = ws * dist;
                    if (dist > 0.0) {
                        const double q = ws / dist;
                        gc = make_float4(static_cast<float>(q * df[0]), static_cast<float>(q * df[1]),
                                         static_cast<float>(q * df[2]), 0.f);
                    }
                }
                d.eatom[i] = e;
                d.fterm[i] = ft;
                d.gFc[i] = gc;
            }
            continue;
        }
        force_out_round<H, K, 0>(WaT, WbT, WcT, D, ND, lane, ti, yv, u, vk, out);
        if (ND > 32) force_out_round<H, K, 32>(WaT, WbT, WcT, D, ND, lane, ti, yv, u, vk, out);
    }
}

// --------------------------------------------------------- head backward --
// Scatter-free reverse pass of both heads (S/model.cpp:318-366) for one
// channel ch per sample, s_ij = fcut (gF_i - gF_j).u_ij on the symmetric CSR:
//   gT_i = S_i Wa[:,ch] + Wb[:,ch] (.) W_i,  S_i = sum_j s_ij,  W_i = sum_j s_ij T_j
//   gh_i = We gE_s + gT_i (.) (1 - T_i^2)
//   dWa[:,ch] += S_i T_i, dWb[:,ch] += T_i (.) W_i / 2, dWc[k,ch] += sum_j (gF_i.u_ij) fcut rbf_ijk,
//   dWe[:,d] += h^L_i gE_s[d]      (per-CTA partials, thread-owned columns)
template <int H, int K, bool kTrain>
struct HeadBody {
    static constexpr bool kFilter = false;
    // train step: s_ij and gF_i.u_ij per edge come staged (k_loss computed them)
    static constexpr int kParts = kTrain ? (kPartPlain | kPartSij) : (kPartGeo | kPartPlain);
    static constexpr bool kBlockHook = false;
    static constexpr bool kPrepare = !kTrain;
    static constexpr int kUnroll = 1;  // block loop unroll (2: the r/rn register roles alternate)
    static constexpr int kBlock = 8;  // edges per block of the walk
    struct Reg {
        float t;
    };
    const Dev& d;
    const float* __restrict__ T;
    const float* __restrict__ hL;
    float* acc;  // smem [3][D][H] + [D][K], this group's
    int a, D, L, pass_ch, first, N;
    bool kv;  // lanes 0..K-1 of warp g % (H/32) carry the rbf-column sums R
    int k;
    int s, ch;
    float Ti, S, W, R;
    float es[8], ed[8];  // per edge of the block: s_ij and gF_i.u_ij
    // loss path (pass_ch < 0): the compact per-atom gradient of k_loss (one head
    // per atom); general upstream: head pass_ch of gF
    __device__ float4 upstream(int j) const {
        if (pass_ch < 0) return __ldg(d.gFc + j);
        const float* gp = d.gF + (static_cast<int64_t>(j) * D + pass_ch) * 3;
        return make_float4(__ldg(gp), __ldg(gp + 1), __ldg(gp + 2), 0.f);
    }
    __device__ void load(const EdgeStage<K>&, int, int j, Reg& r) const {
        r.t = __ldg(T + static_cast<int64_t>(j) * H + a);  // t[L], L >= 1
    }
    // s_ij = fcut (gF_i - gF_j).u_ij is channel-independent: lane u computes edge u
    __device__ void prepare(const EdgeStage<K>& st, int e0) {
        const int lane = threadIdx.x & 31;
        float sij = 0.f, di = 0.f;
        if (lane < 8) {
            const int e = e0 + lane;
            const int i = st.dst[e], j = st.col[e];
            const float4 gv = st.geo[e];
            const float4 gi = i < N ? upstream(i) : make_float4(0.f, 0.f, 0.f, 0.f);  // padding: dst = N
            const float4 gj = upstream(j);
            di = gi.x * gv.x + gi.y * gv.y + gi.z * gv.z;
            const float dj = gj.x * gv.x + gj.y * gv.y + gj.z * gv.z;
            sij = gv.w * (di - dj);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            es[u] = __shfl_sync(0xffffffffu, sij, u);
            ed[u] = __shfl_sync(0xffffffffu, di, u);
        }
    }
    __device__ void edge(const EdgeStage<K>& st, int e, const Reg& r, float, unsigned on) {
        float sv, dv;
        if constexpr (kTrain) {
            const float2 q = st.sij[e];
            sv = q.x, dv = q.y;
        } else {
            sv = es[e & 7], dv = ed[e & 7];
        }
        const float sij = on ? sv : 0.f;
        S += sij;
        W = fmaf(sij, r.t, W);
        if (kv) R = fmaf(on ? dv : 0.f, st.fcp[e * K + k], R);
    }
    // per-atom operands are loaded when the atom begins and used at its end, so
    // their latency hides behind the atom's edges
    float p_wa, p_wb, p_hv, p_ge, p_we, p_gh;
    __device__ void begin(int i) {
        s = d.sample_of[i];
        ch = pass_ch >= 0 ? pass_ch : d.dsidx[s];
        const int row = i;
        Ti = __ldg(T + static_cast<int64_t>(row) * H + a);
        S = W = R = 0.f;
        p_wa = __ldg(d.wfh + a * D + ch);
        p_wb = __ldg(d.wfh + (H + a) * D + ch);
        if (first) {
            p_hv = __ldg(hL + static_cast<int64_t>(row) * H + a);
            p_ge = __ldg(d.gE + static_cast<int64_t>(s) * D + ch);
            p_we = __ldg(d.we + a * D + ch);
        } else {
            p_gh = d.gh[static_cast<int64_t>(i) * H + a];
        }
    }
    __device__ void end(int i) {
        const float gT = S * p_wa + p_wb * W;
        float* ghp = d.gh + static_cast<int64_t>(i) * H + a;
        float gh;
        const float* gE = d.gE + static_cast<int64_t>(s) * D;
        if (first) {
            const float hv = p_hv;
            if (pass_ch < 0) {  // k_loss zeroes every head but the sample's own: same sums, one term
                const float ge = p_ge;
                gh = p_we * ge;
                acc[(2 * D + ch) * H + a] = fmaf(hv, ge, acc[(2 * D + ch) * H + a]);
            } else {
                gh = 0.f;
                for (int dd = 0; dd < D; ++dd) gh = fmaf(d.we[a * D + dd], gE[dd], gh);
                for (int dd = 0; dd < D; ++dd)
                    acc[(2 * D + dd) * H + a] = fmaf(hv, gE[dd], acc[(2 * D + dd) * H + a]);
            }
        } else {
            gh = p_gh;
        }
        *ghp = fmaf(gT, 1.f - Ti * Ti, gh);
        acc[ch * H + a] = fmaf(S, Ti, acc[ch * H + a]);
        acc[(D + ch) * H + a] = fmaf(0.5f * Ti, W, acc[(D + ch) * H + a]);
        if (kv) acc[3 * D * H + ch * K + k] += R;
    }
};

template <int H, int K, bool kTrain>
__global__ void __launch_bounds__(kGroups* H, 1) k_edge_head(Dev d, int pass_ch, int first) {
    EdgeCta<H, K> c = edge_prologue<H, K>(d);
    const int D = d.D;
    const int AW = 3 * D * H + D * K;  // per-group accumulator floats
    float* accs = reinterpret_cast<float*>(c.extra);
    float* acc = accs + c.g * AW;
    for (int e = c.lt; e < AW; e += H) acc[e] = 0.f;
    __syncthreads();
    const int kw = c.g % (H / 32);
    HeadBody<H, K, kTrain> b{d, d.t[d.L], d.h[d.L], acc, c.lt, D, d.L, pass_ch,
                     first, d.hdr->N, (c.lt >> 5) == kw && (c.lt & 31) < K, c.lt & 31};
    walk_edges<H, K>(d, c, b, FilterTc{});
    __syncthreads();
    // combine groups in order; emit the CTA partial in parameter layout:
    //   [ (2H+K) x D force head | H x D energy head ]
    const int NQ = 2 * H + K;
    float* part = d.part_head + static_cast<int64_t>(blockIdx.x) * (NQ + H) * D;
    for (int o = threadIdx.x; o < (NQ + H) * D; o += blockDim.x) {
        const int q = o / D, dd = o % D;
        int src;
        if (q < H) src = dd * H + q;
        else if (q < 2 * H) src = (D + dd) * H + (q - H);
        else if (q < NQ) src = 3 * D * H + dd * K + (q - 2 * H);
        else src = (2 * D + dd) * H + (q - NQ);
        float v = first ? 0.f : part[o];
        for (int gg = 0; gg < kGroups; ++gg) v += accs[gg * AW + src];
        part[o] = v;
    }
}

// ------------------------------------------------------- layer backward --
// Gather form of S/model.cpp:393-418 for layer l:
//   gt_i = sum_j gm_j (.) filter_ij        (filter symmetric in i, j)
//   dWf[a,k] += gm_ia t_ja fcut_ij rbf_ijk (once per edge, thread-owned registers,
//                                           CTA-reduced)
//   gh_i += gt_i (.) (1 - t_i^2)
// The embedding gradient of layer 0 (S/model.cpp:421-424) is k_emb_grad's.
// (A tensor-core dW_f — one M = 128, N = 16, K = 8 MMA per 8-edge block from
// shared-memory G/R tiles — cut the instruction count by a fifth but the
// per-block producer/consumer handshake and the smaller chunk it needs for TMEM
// made the kernel slower; see profiles/README.md.)
template <int H, int K, bool TC, bool kZ>
struct BwdBody {
    static constexpr bool kFilter = TC;
    static constexpr int kParts = kPartPlain | (kZ ? kPartZRow : 0);  // layer 0: Z_j - 1 staged
    static constexpr bool kBlockHook = true;
    static constexpr bool kPrepare = false;
    static constexpr int kUnroll = 1;  // block loop unroll (2: the r/rn register roles alternate)
    static constexpr int kBlock = 8;  // edges per block of the walk
    struct Reg {
        float gm, t;
    };
    const Dev& d;
    const float* __restrict__ tsrc;
    int l, a;
    float w[K];
    uint64_t dw2[K / 2];  // dW_f accumulators as packed fp32 pairs (k, k+1)
    float gmi, gt;
    float gi[8];  // gm of the destination of each edge of the block (0: masked)
    __device__ void load(const EdgeStage<K>& st, int e, int j, Reg& r) const {
        r.gm = __ldg(d.gm + static_cast<int64_t>(j) * H + a);
        const int row = kZ ? st.colz[e] : j;
        r.t = __ldg(tsrc + static_cast<int64_t>(row) * H + a);
    }
    __device__ void edge(const EdgeStage<K>& s, int e, const Reg& r, float f, unsigned on) {
        if constexpr (!TC) f = filter_ffma<K>(w, s, e);
        gt = fmaf(r.gm, on ? f : 0.f, gt);
        if (on) gi[e & 7] = gmi;
    }
    // dWf[a,k] += gm_ia t_ja fcut rbf_k, once per edge (segment-independent),
    // two k per FFMA2
    __device__ void block(const EdgeStage<K>& s, int e0, const Reg (&r)[8], int, int) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint64_t gg = f32x2_splat(gi[u] * r[u].t);
            gi[u] = 0.f;
            const ulonglong2* fr = reinterpret_cast<const ulonglong2*>(s.fcp + (e0 + u) * K);
#pragma unroll
            for (int k4 = 0; k4 < K / 4; ++k4) {
                const ulonglong2 q = fr[k4];
                dw2[2 * k4] = ffma2(gg, q.x, dw2[2 * k4]);
                dw2[2 * k4 + 1] = ffma2(gg, q.y, dw2[2 * k4 + 1]);
            }
        }
    }
    float p_ti, p_gh;  // per-atom operands, loaded at begin() and used at end()
    __device__ void begin(int i) {
        gmi = d.gm[static_cast<int64_t>(i) * H + a];
        gt = 0.f;
        const int row = kZ ? __ldg(d.Z + i) - 1 : i;
        p_ti = __ldg(tsrc + static_cast<int64_t>(row) * H + a);
        p_gh = d.gh[static_cast<int64_t>(i) * H + a];
    }
    __device__ void end(int i) {
        d.gh[static_cast<int64_t>(i) * H + a] = fmaf(gt, 1.f - p_ti * p_ti, p_gh);
    }
};

template <int H, int K, bool kZ>
__global__ void __launch_bounds__(kGroups* H, 1) k_edge_bwd(Dev d, int l) {
    constexpr bool TC = EdgeKernelSmem<H, K>::TC;
    EdgeCta<H, K> c = edge_prologue<H, K>(d);
    float* Wh = reinterpret_cast<float*>(c.extra);
    float* red = Wh + (TC ? 2 * H * K : 0);  // [kGroups][H*K]
    FilterTc ft{};
    if constexpr (TC) {
        ft = filter_setup<H, K>(d, c, l, Wh, Wh + H * K);
    } else {
        __syncthreads();
    }
    BwdBody<H, K, TC, kZ> b{d, kZ ? d.tanh_emb : d.t[l], l, c.lt};
#pragma unroll
    for (int k = 0; k < K; ++k) b.w[k] = TC ? 0.f : d.wf[l][c.lt * K + k];
#pragma unroll
    for (int k = 0; k < K / 2; ++k) b.dw2[k] = 0ull;
#pragma unroll
    for (int u = 0; u < 8; ++u) b.gi[u] = 0.f;
    walk_edges<H, K>(d, c, b, ft);
#pragma unroll
    for (int k = 0; k < K / 2; ++k)
        f32x2_unpack(b.dw2[k], red[c.g * H * K + c.lt * K + 2 * k], red[c.g * H * K + c.lt * K + 2 * k + 1]);
    if constexpr (TC) {
        filter_teardown(c.tslot);
    } else {
        __syncthreads();
    }
    float* part = d.part_wf[l] + static_cast<int64_t>(blockIdx.x) * H * K;
    for (int e = threadIdx.x; e < H * K; e += blockDim.x) {
        float s = 0.f;
        for (int gg = 0; gg < kGroups; ++gg) s += red[gg * H * K + e];
        part[e] = s;
    }
}

}  // namespace lamm_b200
