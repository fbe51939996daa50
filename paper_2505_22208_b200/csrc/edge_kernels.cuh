// edge_kernels.cuh - the four message-passing kernels of the step (forward
// message, force head, head backward, layer backward), sm_100a.
//
// Shape of every kernel: the CSR edge list (grouped by destination atom i, j
// ascending) is cut into Q = gridDim.x * kGroups edge-balanced partitions of
// whole atoms. A CTA runs kGroups independent "groups" of H threads; thread a
// of a group owns feature channel a. A group walks its partition's edges in
// order: edge metadata (j, i, unit/fcut, fcut*rbf) arrives in shared memory in
// 128-edge chunks by TMA bulk copies (cp.async.bulk + mbarrier, double
// buffered); source-atom rows are gathered with one coalesced 4*H-byte load per
// edge across the group (8 edges in flight per thread); the per-destination
// segmented sum is a register accumulation flushed when the destination
// changes. No atomics: parameter-gradient contributions accumulate in
// thread-owned registers / shared memory and leave the kernel as one per-CTA
// partial, summed across CTAs in index order by k_grad_reduce.
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"

namespace lamm_b200 {

constexpr int kGroups = 4;   // independent edge streams per CTA
constexpr int kChunk = 64;   // edges per staged chunk
constexpr int kStages = 2;   // staging double buffer
constexpr int kUnroll = 8;   // gathers in flight per thread

template <int K>
struct EdgeStage {
    int32_t col[kChunk];
    int32_t dst[kChunk];
    float4 geo[kChunk];
    float fcrbf[kChunk * K];
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
__device__ __forceinline__ void group_sync(int g, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(nthreads) : "memory");
}

// Walks the edges of atoms [lo, hi) for one group. Body provides:
//   struct Reg;                                  per-edge gathered registers
//   void load(const EdgeStage<K>&, int e, Reg&); issue the edge's gathers
//   void edge(const EdgeStage<K>&, int e, const Reg&);
//   void begin(int i); void end(int i);          destination-atom brackets
template <int H, int K, class Body>
__device__ __forceinline__ void walk_edges(const Dev& d, EdgeStage<K>* st, uint64_t* bar, int g, int lt, int lo,
                                           int hi, Body& body) {
    if (lo >= hi) return;
    const int e0 = d.row_ptr[lo], e1 = d.row_ptr[hi];
    int cur = lo;
    body.begin(cur);
    if (e1 > e0) {
        const int base = e0 & ~3;  // 16-byte aligned chunk origin
        const int nchunks = (e1 - base + kChunk - 1) / kChunk;
        auto issue = [&](int k) {
            const int cb = base + k * kChunk;
            const int n = min(kChunk, ((e1 - cb) + 3) & ~3);
            EdgeStage<K>& s = st[k % kStages];
            uint64_t* b = &bar[k % kStages];
            mbar_expect_tx(b, static_cast<uint32_t>(n * (8 + 16 + 4 * K)));
            bulk_g2s(s.col, d.col + cb, 4 * n, b);
            bulk_g2s(s.dst, d.dst + cb, 4 * n, b);
            bulk_g2s(s.geo, d.geo + cb, 16 * n, b);
            bulk_g2s(s.fcrbf, d.rbf + static_cast<int64_t>(cb) * K, 4 * K * n, b);
        };
        if (lt == 0) {
            issue(0);
            if (nchunks > 1) issue(1);
        }
        for (int k = 0; k < nchunks; ++k) {
            mbar_wait(&bar[k % kStages], (k / kStages) & 1);
            const EdgeStage<K>& s = st[k % kStages];
            const int cb = base + k * kChunk;
            const int ea = max(cb, e0) - cb, eb = min(cb + kChunk, e1) - cb;
            for (int el = ea; el < eb; el += kUnroll) {
                typename Body::Reg r[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
                    if (el + u < eb) body.load(s, el + u, r[u]);
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    if (el + u < eb) {
                        const int i = s.dst[el + u];
                        while (cur < i) {
                            body.end(cur);
                            ++cur;
                            body.begin(cur);
                        }
                        body.edge(s, el + u, r[u]);
                    }
                }
            }
            group_sync(g, H);  // every thread is done with this stage
            if (lt == 0 && k + kStages < nchunks) issue(k + kStages);
        }
    }
    body.end(cur);
    for (int i = cur + 1; i < hi; ++i) {
        body.begin(i);
        body.end(i);
    }
}

// Shared-memory layout common to the edge kernels: per group kStages staged
// chunks + barriers, then the kernel's own region.
template <int K>
struct EdgeSmem {
    static constexpr size_t stage_bytes = sizeof(EdgeStage<K>) * kStages * kGroups;
    static constexpr size_t bar_bytes = 16 * kStages * kGroups;
    static constexpr size_t extra_offset = stage_bytes + bar_bytes;
};

template <int H, int K>
struct EdgeCta {
    EdgeStage<K>* st;
    uint64_t* bar;
    char* extra;
    int g, lt, lo, hi;
};

// Common prologue: carve shared memory, init barriers, find the partition.
template <int H, int K>
__device__ __forceinline__ EdgeCta<H, K> edge_prologue(const Dev& d) {
    extern __shared__ __align__(128) unsigned char lamm_edge_smem[];
    EdgeCta<H, K> c;
    c.g = threadIdx.x / H;
    c.lt = threadIdx.x % H;
    c.st = reinterpret_cast<EdgeStage<K>*>(lamm_edge_smem) + c.g * kStages;
    c.bar = reinterpret_cast<uint64_t*>(lamm_edge_smem + EdgeSmem<K>::stage_bytes) + c.g * kStages;
    c.extra = reinterpret_cast<char*>(lamm_edge_smem + EdgeSmem<K>::extra_offset);
    if (c.lt == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&c.bar[s], 1);
        mbar_fence_init();
    }
    const int q = blockIdx.x * kGroups + c.g;  // partitions cut by k_scan
    c.lo = d.part_lo[q];
    c.hi = d.part_lo[q + 1];
    __syncthreads();
    return c;
}

// ---------------------------------------------------------------- message --
// m_i[a] = sum_j t_j[a] * sum_k Wf[a,k] fcut_ij rbf_ijk ; mu_i = tanh(m_i)   (S/model.cpp:78-93)
template <int H, int K>
struct MessageBody {
    struct Reg {
        float t;
    };
    const Dev& d;
    const float* __restrict__ tsrc;
    int l, a;
    float w[K];
    float m;
    __device__ void load(const EdgeStage<K>& s, int e, Reg& r) const {
        const int j = s.col[e];
        const int row = l == 0 ? __ldg(d.Z + j) - 1 : j;
        r.t = __ldg(tsrc + static_cast<int64_t>(row) * H + a);
    }
    __device__ void edge(const EdgeStage<K>& s, int e, const Reg& r) {
        const float4* fr = reinterpret_cast<const float4*>(s.fcrbf + e * K);
        float f = 0.f;
#pragma unroll
        for (int k4 = 0; k4 < K / 4; ++k4) {
            const float4 q = fr[k4];
            f = fmaf(w[4 * k4], q.x, f);
            f = fmaf(w[4 * k4 + 1], q.y, f);
            f = fmaf(w[4 * k4 + 2], q.z, f);
            f = fmaf(w[4 * k4 + 3], q.w, f);
        }
        m = fmaf(r.t, f, m);
    }
    __device__ void begin(int) { m = 0.f; }
    __device__ void end(int i) { d.mu[l][static_cast<int64_t>(i) * H + a] = tanhf(m); }
};

template <int H, int K>
__global__ void __launch_bounds__(kGroups* H) k_edge_message(Dev d, int l) {
    EdgeCta<H, K> c = edge_prologue<H, K>(d);
    MessageBody<H, K> b{d, l == 0 ? d.tanh_emb : d.t[l], l, c.lt};
#pragma unroll
    for (int k = 0; k < K; ++k) b.w[k] = d.wf[l][c.lt * K + k];
    walk_edges<H, K>(d, c.st, c.bar, c.g, c.lt, c.lo, c.hi, b);
}

// ------------------------------------------------------------ force head --
// F_i^d = sum_j [ (A_i^d + A_j^d) fcut + sum_k Wc[k,d] fcut rbf_k ] u_ij
//       + sum_a Wb[a,d] T_ia Y_i[a],  Y_i[a] = sum_j T_ja fcut_ij u_ij     (S/model.cpp:223-253)
// Thread lt < 3D also owns output (d, x) = (lt / 3, lt % 3) of the scalar part.
template <int H, int K>
struct ForceBody {
    struct Reg {
        float t, aj;
    };
    const Dev& d;
    const float* __restrict__ T;
    const float* WbT;  // smem [D][H]
    const float* Wc;   // smem [K][D]
    float* red;        // smem [H/32][32] group reduction scratch
    int a, g, D, ND, L;
    int dd, xx;
    float Ti, Y0, Y1, Y2, Fs, Ai;
    __device__ void load(const EdgeStage<K>& s, int e, Reg& r) const {
        const int j = s.col[e];
        const int row = L > 0 ? j : __ldg(d.Z + j) - 1;
        r.t = __ldg(T + static_cast<int64_t>(row) * H + a);
        r.aj = a < ND ? __ldg(d.A + static_cast<int64_t>(j) * D + dd) : 0.f;
    }
    __device__ void edge(const EdgeStage<K>& s, int e, const Reg& r) {
        const float4 gv = s.geo[e];
        const float tf = r.t * gv.w;
        Y0 = fmaf(tf, gv.x, Y0);
        Y1 = fmaf(tf, gv.y, Y1);
        Y2 = fmaf(tf, gv.z, Y2);
        if (a < ND) {
            float wc = 0.f;
            const float* fr = s.fcrbf + e * K;
#pragma unroll
            for (int k = 0; k < K; ++k) wc = fmaf(Wc[k * D + dd], fr[k], wc);
            const float ux = xx == 0 ? gv.x : (xx == 1 ? gv.y : gv.z);
            Fs = fmaf(fmaf(Ai + r.aj, gv.w, wc), ux, Fs);
        }
    }
    __device__ void begin(int i) {
        const int row = L > 0 ? i : __ldg(d.Z + i) - 1;
        Ti = __ldg(T + static_cast<int64_t>(row) * H + a);
        Y0 = Y1 = Y2 = Fs = 0.f;
        Ai = a < ND ? d.A[static_cast<int64_t>(i) * D + dd] : 0.f;
    }
    __device__ void end(int i) {
        const int lane = a & 31, warp = a >> 5;
        const float y[3] = {Y0, Y1, Y2};
        float total = 0.f;
        for (int r0 = 0; r0 < ND; r0 += 32) {
            float v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int idx = r0 + k;
                float s = 0.f;
                if (idx < ND) s = WbT[(idx / 3) * H + a] * Ti * y[idx % 3];
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
            red[warp * 32 + lane] = v[0];
            group_sync(g, H);
            if (a >= r0 && a < r0 + 32 && a < ND) {
                float t = 0.f;
                for (int w = 0; w < H / 32; ++w) t += red[w * 32 + (a - r0)];
                total = t;
            }
            group_sync(g, H);
        }
        if (a < ND) d.F[static_cast<int64_t>(i) * ND + a] = Fs + total;
    }
};

template <int H, int K>
__global__ void __launch_bounds__(kGroups* H) k_edge_force(Dev d) {
    EdgeCta<H, K> c = edge_prologue<H, K>(d);
    const int D = d.D;
    float* WbT = reinterpret_cast<float*>(c.extra);  // [D][H]
    float* Wc = WbT + D * H;                          // [K][D]
    float* red = Wc + K * D + c.g * H;                // [kGroups][H]
    for (int idx = threadIdx.x; idx < D * H; idx += blockDim.x) {
        const int dd = idx / H, a = idx % H;
        WbT[idx] = d.wfh[(H + a) * D + dd];
    }
    for (int idx = threadIdx.x; idx < K * D; idx += blockDim.x) Wc[idx] = d.wfh[2 * H * D + idx];
    __syncthreads();
    ForceBody<H, K> b{d, d.L > 0 ? d.t[d.L] : d.tanh_emb, WbT, Wc, red, c.lt, c.g, D, 3 * D, d.L};
    b.dd = c.lt / 3, b.xx = c.lt % 3;
    walk_edges<H, K>(d, c.st, c.bar, c.g, c.lt, c.lo, c.hi, b);
}

// --------------------------------------------------------- head backward --
// Scatter-free reverse pass of both heads (S/model.cpp:318-366) for one
// channel ch per sample, s_ij = fcut (gF_i - gF_j).u_ij on the symmetric CSR:
//   gT_i = S_i Wa[:,ch] + Wb[:,ch] (.) W_i,  S_i = sum_j s_ij,  W_i = sum_j s_ij T_j
//   gh_i = We gE_s + gT_i (.) (1 - T_i^2)
//   dWa[:,ch] += S_i T_i, dWb[:,ch] += T_i (.) W_i / 2, dWc[k,ch] += sum_j (gF_i.u_ij) fcut rbf_ijk,
//   dWe[:,d] += h^L_i gE_s[d]      (per-CTA partials, thread-owned columns)
template <int H, int K>
struct HeadBody {
    struct Reg {
        float t, g0, g1, g2;
    };
    const Dev& d;
    const float* __restrict__ T;
    const float* __restrict__ hL;
    float* acc;  // smem [3][D][H] + [D][K], this group's
    int a, D, L, pass_ch, first;
    int s, ch;
    float Ti, S, W, R, gf0, gf1, gf2;
    __device__ void load(const EdgeStage<K>& st, int e, Reg& r) const {
        const int j = st.col[e];
        const int row = L > 0 ? j : __ldg(d.Z + j) - 1;
        r.t = __ldg(T + static_cast<int64_t>(row) * H + a);
        // channel of the edge's own sample (the unrolled window may run ahead of begin())
        const int chj = pass_ch >= 0 ? pass_ch : __ldg(d.chan + j);
        const float* gp = d.gF + (static_cast<int64_t>(j) * D + chj) * 3;
        r.g0 = __ldg(gp), r.g1 = __ldg(gp + 1), r.g2 = __ldg(gp + 2);
    }
    __device__ void edge(const EdgeStage<K>& st, int e, const Reg& r) {
        const float4 gv = st.geo[e];
        const float di = gf0 * gv.x + gf1 * gv.y + gf2 * gv.z;
        const float dj = r.g0 * gv.x + r.g1 * gv.y + r.g2 * gv.z;
        const float sij = gv.w * (di - dj);
        S += sij;
        W = fmaf(sij, r.t, W);
        if (a < K) R = fmaf(di, st.fcrbf[e * K + a], R);
    }
    __device__ void begin(int i) {
        s = d.sample_of[i];
        ch = pass_ch >= 0 ? pass_ch : d.dsidx[s];
        const int row = L > 0 ? i : __ldg(d.Z + i) - 1;
        Ti = __ldg(T + static_cast<int64_t>(row) * H + a);
        const float* gp = d.gF + (static_cast<int64_t>(i) * D + ch) * 3;
        gf0 = gp[0], gf1 = gp[1], gf2 = gp[2];
        S = W = R = 0.f;
    }
    __device__ void end(int i) {
        const float wa = d.wfh[a * D + ch], wb = d.wfh[(H + a) * D + ch];
        const float gT = S * wa + wb * W;
        float* ghp = d.gh + static_cast<int64_t>(i) * H + a;
        float gh;
        const float* gE = d.gE + static_cast<int64_t>(s) * D;
        if (first) {
            gh = 0.f;
            for (int dd = 0; dd < D; ++dd) gh = fmaf(d.we[a * D + dd], gE[dd], gh);
            const int row = L > 0 ? i : __ldg(d.Z + i) - 1;
            const float hv = hL[static_cast<int64_t>(row) * H + a];
            for (int dd = 0; dd < D; ++dd) acc[(2 * D + dd) * H + a] = fmaf(hv, gE[dd], acc[(2 * D + dd) * H + a]);
        } else {
            gh = *ghp;
        }
        *ghp = fmaf(gT, 1.f - Ti * Ti, gh);
        acc[ch * H + a] = fmaf(S, Ti, acc[ch * H + a]);
        acc[(D + ch) * H + a] = fmaf(0.5f * Ti, W, acc[(D + ch) * H + a]);
        if (a < K) acc[3 * D * H + ch * K + a] += R;
    }
};

template <int H, int K>
__global__ void __launch_bounds__(kGroups* H) k_edge_head(Dev d, int pass_ch, int first) {
    EdgeCta<H, K> c = edge_prologue<H, K>(d);
    const int D = d.D;
    const int AW = 3 * D * H + D * K;  // per-group accumulator floats
    float* accs = reinterpret_cast<float*>(c.extra);
    float* acc = accs + c.g * AW;
    for (int e = c.lt; e < AW; e += H) acc[e] = 0.f;
    group_sync(c.g, H);
    HeadBody<H, K> b{d, d.L > 0 ? d.t[d.L] : d.tanh_emb, d.L > 0 ? d.h[d.L] : d.emb, acc, c.lt, D, d.L, pass_ch,
                     first};
    walk_edges<H, K>(d, c.st, c.bar, c.g, c.lt, c.lo, c.hi, b);
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
//   gt_i = sum_j gm_j (.) filter_ij ;  dWf[a,k] += gm_ia t_ja fcut_ij rbf_ijk ;
//   gh_i += gt_i (.) (1 - t_i^2) ; on layer 0 also dE[Z_i] += gh_i (S/model.cpp:421-424).
template <int H, int K>
struct BwdBody {
    struct Reg {
        float gm, t;
    };
    const Dev& d;
    const float* __restrict__ tsrc;
    float* emb_acc;  // smem [slots][H] (layer 0), this group's
    int l, a;
    float w[K], dw[K];
    float gmi, gt;
    __device__ void load(const EdgeStage<K>& s, int e, Reg& r) const {
        const int j = s.col[e];
        r.gm = __ldg(d.gm + static_cast<int64_t>(j) * H + a);
        const int row = l == 0 ? __ldg(d.Z + j) - 1 : j;
        r.t = __ldg(tsrc + static_cast<int64_t>(row) * H + a);
    }
    __device__ void edge(const EdgeStage<K>& s, int e, const Reg& r) {
        const float4* fr = reinterpret_cast<const float4*>(s.fcrbf + e * K);
        float q[K];
#pragma unroll
        for (int k4 = 0; k4 < K / 4; ++k4) {
            const float4 v = fr[k4];
            q[4 * k4] = v.x, q[4 * k4 + 1] = v.y, q[4 * k4 + 2] = v.z, q[4 * k4 + 3] = v.w;
        }
        float f = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) f = fmaf(w[k], q[k], f);
        gt = fmaf(r.gm, f, gt);
        const float gg = gmi * r.t;
#pragma unroll
        for (int k = 0; k < K; ++k) dw[k] = fmaf(gg, q[k], dw[k]);
    }
    __device__ void begin(int i) {
        gmi = d.gm[static_cast<int64_t>(i) * H + a];
        gt = 0.f;
    }
    __device__ void end(int i) {
        const int row = l == 0 ? __ldg(d.Z + i) - 1 : i;
        const float ti = __ldg(tsrc + static_cast<int64_t>(row) * H + a);
        float* ghp = d.gh + static_cast<int64_t>(i) * H + a;
        const float gh = fmaf(gt, 1.f - ti * ti, *ghp);
        *ghp = gh;
        if (l == 0) emb_acc[d.zslot[i] * H + a] += gh;
    }
};

template <int H, int K>
__global__ void __launch_bounds__(kGroups* H) k_edge_bwd(Dev d, int l, int slot_cap) {
    EdgeCta<H, K> c = edge_prologue<H, K>(d);
    float* red = reinterpret_cast<float*>(c.extra);          // [kGroups][H*K]
    float* emb = red + kGroups * H * K;                      // [kGroups][slot_cap][H]
    const int ns = d.hdr->nslots;
    if (l == 0)
        for (int e = c.lt; e < ns * H; e += H) emb[c.g * slot_cap * H + e] = 0.f;
    group_sync(c.g, H);
    BwdBody<H, K> b{d, l == 0 ? d.tanh_emb : d.t[l], emb + c.g * slot_cap * H, l, c.lt};
#pragma unroll
    for (int k = 0; k < K; ++k) b.w[k] = d.wf[l][c.lt * K + k], b.dw[k] = 0.f;
    walk_edges<H, K>(d, c.st, c.bar, c.g, c.lt, c.lo, c.hi, b);
#pragma unroll
    for (int k = 0; k < K; ++k) red[c.g * H * K + c.lt * K + k] = b.dw[k];
    __syncthreads();
    float* part = d.part_wf[l] + static_cast<int64_t>(blockIdx.x) * H * K;
    for (int e = threadIdx.x; e < H * K; e += blockDim.x) {
        float s = 0.f;
        for (int gg = 0; gg < kGroups; ++gg) s += red[gg * H * K + e];
        part[e] = s;
    }
    if (l == 0) {
        float* pe = d.part_emb + static_cast<int64_t>(blockIdx.x) * ns * H;
        for (int e = threadIdx.x; e < ns * H; e += blockDim.x) {
            float s = 0.f;
            for (int gg = 0; gg < kGroups; ++gg) s += emb[gg * slot_cap * H + e];
            pe[e] = s;
        }
    }
}

}  // namespace lamm_b200
