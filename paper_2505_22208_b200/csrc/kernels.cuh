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
//   k_nbr_* ......... S/core.cpp:30-48  (bit-exact fp64 pair test, i-major, j ascending)
//   k_message ....... S/model.cpp:78-92 (filter = W_f rbf fcut; m_i = sum_j t_j * filter)
//   k_update ........ S/model.cpp:93-102 (h' = h + W_u tanh(m)), + :208-218 energy head
//   k_force ......... S/model.cpp:223-253 (pair force head; A_i + A_j split)
//   k_energy/k_loss . S/loss.cpp:140-213 (Eq. 5, per-rank mask denominators)
//   k_head_bwd ...... S/model.cpp:318-366 (scatter-free: gather over the symmetric CSR)
//   k_bwd_gemm ...... S/model.cpp:377-390 (dW_u, gm)
//   k_bwd_edge ...... S/model.cpp:393-418 (gt_l gather, dW_f)
//   k_embed_grad .... S/model.cpp:421-424
//   k_opt_* ......... S/trainer.cpp:319-327 + RmsOptimizer :37-53
//
// Determinism: no floating-point atomics. Parameter gradients are reduced into
// per-CTA partials in a fixed order and summed across CTAs in index order by
// k_grad_reduce; the grid sizes are fixed per device, so a step is bit-for-bit
// reproducible run to run.
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"

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

__global__ void __launch_bounds__(128) k_prep(Dev d, BatchArrays out) {
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
    __shared__ double mean[3];
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
    }
}

// ------------------------------------------------------- neighbour list ---
// Bit-exact with S/core.cpp:40-43: d = p_i - p_j, r = sqrt((dx*dx + dy*dy) + dz*dz)
// with every operation individually rounded (no FMA contraction), r < cutoff.
__device__ __forceinline__ double pair_dist(double xi, double yi, double zi, double xj, double yj, double zj,
                                            double& dx, double& dy, double& dz) {
    dx = __dsub_rn(xi, xj);
    dy = __dsub_rn(yi, yj);
    dz = __dsub_rn(zi, zj);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

// Warp per destination atom i; lanes sweep the sample's atoms j in order and
// count with ballot/popc.
__global__ void __launch_bounds__(256) k_nbr_count(Dev d) {
    const int N = d.hdr->N;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
        const int s = d.sample_of[i];
        const int lo = static_cast<int>(d.atom_ptr[s]), hi = static_cast<int>(d.atom_ptr[s + 1]);
        const double xi = d.x[i], yi = d.y[i], zi = d.z[i];
        int cnt = 0;
        for (int j0 = lo; j0 < hi; j0 += 32) {
            const int j = j0 + lane;
            bool in = false;
            if (j < hi && j != i) {
                double dx, dy, dz;
                in = pair_dist(xi, yi, zi, d.x[j], d.y[j], d.z[j], dx, dy, dz) < d.rc;
            }
            cnt += __popc(__ballot_sync(0xffffffffu, in));
        }
        if (lane == 0) d.cnt[i] = cnt;
    }
}

// Single-CTA exclusive scan of the per-atom pair counts into row_ptr; writes P
// and the capacity-overflow flag.
__global__ void __launch_bounds__(1024) k_scan(Dev d) {
    __shared__ int warp_tot[32];
    const int N = d.hdr->N;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int per = (N + 1023) / 1024;
    const int b = min(N, t * per), e = min(N, b + per);
    int s = 0;
    for (int k = b; k < e; ++k) s += d.cnt[k];
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int w = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += v;
        }
        warp_tot[lane] = w;
    }
    __syncthreads();
    int run = incl - s + (wid > 0 ? warp_tot[wid - 1] : 0);
    for (int k = b; k < e; ++k) {
        d.row_ptr[k] = run;
        run += d.cnt[k];
    }
    if (t == 1023) {
        d.row_ptr[N] = run;
        d.hdr->P = run;
        d.hdr->overflow = static_cast<int64_t>(run) > d.Pcap ? 1 : 0;
    }
}

// Same sweep as k_nbr_count; lanes that hold a neighbour compact into the CSR
// row with popc(ballot & lanes_below). Edge geometry is computed in fp64 and
// rounded once: unit (1/r)*d (S/core.cpp:43), fcut (S/model.cpp:17), Gaussians
// (S/model.cpp:20-27).
template <int K>
__global__ void __launch_bounds__(256) k_nbr_fill(Dev d) {
    if (d.hdr->overflow) return;
    const int N = d.hdr->N;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const double width = d.rc / static_cast<double>(K - 1);
    const double inv = 1.0 / (2.0 * width * width);
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
        const int s = d.sample_of[i];
        const int lo = static_cast<int>(d.atom_ptr[s]), hi = static_cast<int>(d.atom_ptr[s + 1]);
        const double xi = d.x[i], yi = d.y[i], zi = d.z[i];
        int base = d.row_ptr[i];
        for (int j0 = lo; j0 < hi; j0 += 32) {
            const int j = j0 + lane;
            bool in = false;
            double dx = 0, dy = 0, dz = 0, r = 0;
            if (j < hi && j != i) {
                r = pair_dist(xi, yi, zi, d.x[j], d.y[j], d.z[j], dx, dy, dz);
                in = r < d.rc;
            }
            const unsigned mask = __ballot_sync(0xffffffffu, in);
            if (in) {
                const int p = base + __popc(mask & ((1u << lane) - 1u));
                d.col[p] = j;
                const double sc = __ddiv_rn(1.0, r);
                const double ux = __dmul_rn(sc, dx), uy = __dmul_rn(sc, dy), uz = __dmul_rn(sc, dz);
                const double fc = 0.5 * (cos(kPiD * r / d.rc) + 1.0);
                d.geo[p] = make_float4(static_cast<float>(ux), static_cast<float>(uy), static_cast<float>(uz),
                                       static_cast<float>(fc));
                float rb[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double dd = r - width * static_cast<double>(k);
                    rb[k] = static_cast<float>(exp(-dd * dd * inv));
                }
                float4* dst = reinterpret_cast<float4*>(d.rbf + static_cast<int64_t>(p) * K);
#pragma unroll
                for (int k = 0; k < K / 4; ++k) dst[k] = make_float4(rb[4 * k], rb[4 * k + 1], rb[4 * k + 2], rb[4 * k + 3]);
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

// --------------------------------------------------------------- encoder ---
// Message of layer l, warp per destination atom: lane owns channels
// [lane*C, lane*C+C), keeps its C x K slice of W_f in registers, walks the
// atom's CSR row (edges contiguous, j ascending), gathers t_j rows with one
// coalesced vector load per lane, and reduces in registers (no atomics).
// Writes mu_l = tanh(m_l).
template <int H, int K>
__global__ void __launch_bounds__(256) k_message(Dev d, int l) {
    constexpr int C = H / 32;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    float w[C][K];
    const float* __restrict__ wf = d.wf[l];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int k = 0; k < K; ++k) w[c][k] = wf[(lane * C + c) * K + k];
    const float* __restrict__ tsrc = l == 0 ? d.tanh_emb : d.t[l];
    const int N = d.hdr->N;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
        const int p0 = d.row_ptr[i], p1 = d.row_ptr[i + 1];
        float m[C];
#pragma unroll
        for (int c = 0; c < C; ++c) m[c] = 0.f;
#pragma unroll 2
        for (int p = p0; p < p1; ++p) {
            const int j = __ldg(d.col + p);
            const float fc = __ldg(&d.geo[p].w);
            float rb[K];
            load_rbf<K>(d.rbf + static_cast<int64_t>(p) * K, rb);
            const int jrow = l == 0 ? __ldg(d.Z + j) - 1 : j;
            const VecF<C> tj = ldv<C>(tsrc + static_cast<int64_t>(jrow) * H + lane * C);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < K; ++k) acc = fmaf(w[c][k], rb[k], acc);
                m[c] = fmaf(tj.v[c], acc * fc, m[c]);
            }
        }
        VecF<C> o;
#pragma unroll
        for (int c = 0; c < C; ++c) o.v[c] = tanhf(m[c]);
        stv<C>(d.mu[l] + static_cast<int64_t>(i) * H + lane * C, o);
    }
}

// Update of layer l: h_{l+1} = h_l + mu_l W_u^T as a persistent tile GEMM
// (32 atoms x H per tile, W_u^T staged once per CTA in shared memory), fused
// epilogue writes h_{l+1} and t_{l+1} = tanh(h_{l+1}). On the last layer the
// epilogue also produces the per-atom energy e_i[d] = W_e^T h^L_i and the
// force-head split A_i[d] = W_fh[0:H]^T t^L_i.
template <int H>
__global__ void __launch_bounds__(256) k_update(Dev d, int l, int last) {
    constexpr int C = H / 32, TM = 32, RPW = TM / 8;
    float* sm = dyn_smem<float>();
    float* WuT = sm;           // [H][H], WuT[a][b] = W_u[b][a]
    float* tile = sm + H * H;  // [TM][H]
    float* tile2 = tile + TM * H;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* __restrict__ wu = d.wu[l];
    for (int idx = tid; idx < H * H; idx += blockDim.x) {
        const int a = idx / H, b = idx % H;
        WuT[idx] = wu[b * H + a];
    }
    const int N = d.hdr->N, D = d.D;
    const int ntiles = (N + TM - 1) / TM;
    __syncthreads();
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const int base = ti * TM;
        for (int idx = tid * 4; idx < TM * H; idx += blockDim.x * 4) {
            const int r = idx / H, atom = base + r;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (atom < N) v = *reinterpret_cast<const float4*>(d.mu[l] + static_cast<int64_t>(atom) * H + idx % H);
            *reinterpret_cast<float4*>(tile + idx) = v;
        }
        __syncthreads();
        float acc[RPW][C];
#pragma unroll
        for (int r = 0; r < RPW; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[r][c] = 0.f;
        const int r0 = warp * RPW;
#pragma unroll 4
        for (int a = 0; a < H; ++a) {
            const VecF<C> wv = ldv<C>(WuT + a * H + lane * C);
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                const float mv = tile[(r0 + r) * H + a];
#pragma unroll
                for (int c = 0; c < C; ++c) acc[r][c] = fmaf(mv, wv.v[c], acc[r][c]);
            }
        }
        if (last) __syncthreads();  // tile is reused for h^L below
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int atom = base + r0 + r;
            if (atom >= N) continue;
            const float* hp = l == 0 ? d.emb + static_cast<int64_t>(__ldg(d.Z + atom) - 1) * H
                                     : d.h[l] + static_cast<int64_t>(atom) * H;
            const VecF<C> hv = ldv<C>(hp + lane * C);
            VecF<C> hn, tn;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                hn.v[c] = hv.v[c] + acc[r][c];
                tn.v[c] = tanhf(hn.v[c]);
            }
            stv<C>(d.h[l + 1] + static_cast<int64_t>(atom) * H + lane * C, hn);
            stv<C>(d.t[l + 1] + static_cast<int64_t>(atom) * H + lane * C, tn);
            if (last) {
                stv<C>(tile + (r0 + r) * H + lane * C, hn);
                stv<C>(tile2 + (r0 + r) * H + lane * C, tn);
            }
        }
        if (last) {
            __syncthreads();
            for (int o = tid; o < TM * D * 2; o += blockDim.x) {
                const int r = o / (2 * D), q = o % (2 * D), which = q / D, dd = q % D;
                const int atom = base + r;
                if (atom >= N) continue;
                const float* src = (which ? tile2 : tile) + r * H;
                const float* W = which ? d.wfh : d.we;
                float s = 0.f;
#pragma unroll 8
                for (int a = 0; a < H; ++a) s = fmaf(src[a], __ldg(W + a * D + dd), s);
                (which ? d.A : d.e_atom)[static_cast<int64_t>(atom) * D + dd] = s;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ force head ---
// In-warp reduce-scatter of 32 per-lane values: after 31 shuffles lane k holds
// the warp sum of value k.
__device__ __forceinline__ float reduce_scatter32(float (&v)[32], int lane) {
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
    return v[0];
}

// F_i^d = sum_j w_ijd fcut_ij u_ij with w_ijd = A_id + A_jd + sum_a Wb[a,d] T_ia T_ja
// + sum_k Wc[k,d] rbf_ijk. Re-associated per destination atom: the Wb term is
// sum_a Wb[a,d] T_ia Y_i[a] with Y_i = sum_j T_j fcut u (accumulated per lane in
// registers), so the only per-edge work is one T_j gather plus O(K + D) scalar
// flops; the 3D outputs are produced by one reduce-scatter per atom.
template <int H, int K>
__global__ void __launch_bounds__(256) k_force(Dev d) {
    constexpr int C = H / 32;
    float* sm = dyn_smem<float>();
    const int D = d.D, ND = 3 * D;
    float* WbT = sm;              // [D][H]
    float* Wc = sm + D * H;       // [K][D]
    for (int idx = threadIdx.x; idx < D * H; idx += blockDim.x) {
        const int dd = idx / H, a = idx % H;
        WbT[idx] = d.wfh[(H + a) * D + dd];
    }
    for (int idx = threadIdx.x; idx < K * D; idx += blockDim.x) Wc[idx] = d.wfh[2 * H * D + idx];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int N = d.hdr->N, L = d.L;
    const float* __restrict__ T = L > 0 ? d.t[L] : d.tanh_emb;
    const int R = (ND + 31) / 32;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
        const int irow = L > 0 ? i : __ldg(d.Z + i) - 1;
        const VecF<C> Ti = ldv<C>(T + static_cast<int64_t>(irow) * H + lane * C);
        float Ai[3], Fs[3];
        int ddl[3], xl[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int idx = 32 * r + lane;
            ddl[r] = idx / 3, xl[r] = idx % 3;
            Ai[r] = (r < R && idx < ND) ? d.A[static_cast<int64_t>(i) * D + ddl[r]] : 0.f;
            Fs[r] = 0.f;
        }
        float Y[C][3];
#pragma unroll
        for (int c = 0; c < C; ++c) Y[c][0] = Y[c][1] = Y[c][2] = 0.f;
        const int p0 = d.row_ptr[i], p1 = d.row_ptr[i + 1];
        for (int p = p0; p < p1; ++p) {
            const int j = __ldg(d.col + p);
            const float4 g = __ldg(d.geo + p);
            float rb[K];
            load_rbf<K>(d.rbf + static_cast<int64_t>(p) * K, rb);
            const int jrow = L > 0 ? j : __ldg(d.Z + j) - 1;
            const VecF<C> Tj = ldv<C>(T + static_cast<int64_t>(jrow) * H + lane * C);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const float tf = Tj.v[c] * g.w;
                Y[c][0] = fmaf(tf, g.x, Y[c][0]);
                Y[c][1] = fmaf(tf, g.y, Y[c][1]);
                Y[c][2] = fmaf(tf, g.z, Y[c][2]);
            }
            const float u[3] = {g.x, g.y, g.z};
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const int idx = 32 * r + lane;
                if (r < R && idx < ND) {
                    float w = Ai[r] + __ldg(d.A + static_cast<int64_t>(j) * D + ddl[r]);
#pragma unroll
                    for (int k = 0; k < K; ++k) w = fmaf(Wc[k * D + ddl[r]], rb[k], w);
                    const float ux = xl[r] == 0 ? u[0] : (xl[r] == 1 ? u[1] : u[2]);
                    Fs[r] = fmaf(w * g.w, ux, Fs[r]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            if (r >= R) break;
            float v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int idx = 32 * r + k;
                float s = 0.f;
                if (idx < ND) {
                    const int dd = idx / 3, x = idx % 3;
                    const VecF<C> wb = ldv<C>(WbT + dd * H + lane * C);
#pragma unroll
                    for (int c = 0; c < C; ++c) s = fmaf(wb.v[c] * Ti.v[c], Y[c][x], s);
                }
                v[k] = s;
            }
            const float tot = reduce_scatter32(v, lane);
            const int idx = 32 * r + lane;
            if (idx < ND) d.F[static_cast<int64_t>(i) * ND + idx] = Fs[r] + tot;
        }
    }
}

// ---------------------------------------------------------------- energy ---
// Per-sample energies for every head, E_s^d = sum_{i in s} e_i^d, in fp64.
__global__ void __launch_bounds__(128) k_energy(Dev d) {
    double* red = dyn_smem<double>();  // [D][128]
    const int B = d.hdr->B, D = d.D;
    for (int s = blockIdx.x; s < B; s += gridDim.x) {
        const int64_t lo = d.atom_ptr[s], hi = d.atom_ptr[s + 1];
        for (int dd = 0; dd < D; ++dd) red[dd * 128 + threadIdx.x] = 0.0;
        for (int64_t a = lo + threadIdx.x; a < hi; a += 128)
            for (int dd = 0; dd < D; ++dd) red[dd * 128 + threadIdx.x] += static_cast<double>(d.e_atom[a * D + dd]);
        __syncthreads();
        for (int o = 64; o > 0; o >>= 1) {
            if (threadIdx.x < o)
                for (int dd = 0; dd < D; ++dd) red[dd * 128 + threadIdx.x] += red[dd * 128 + threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x < D) d.Epred[static_cast<int64_t>(s) * D + threadIdx.x] = red[threadIdx.x * 128];
        __syncthreads();
    }
}

// ------------------------------------------------------------------ loss ---
// Eq. (5) with the per-rank denominators sum m_E, sum m_F (S/loss.cpp:175-212):
// block per sample computes its energy/force terms and writes d(loss)/d(pred)
// for the selected head d_s only (every other channel is zeroed).
__global__ void __launch_bounds__(128) k_loss(Dev d) {
    __shared__ double red[128];
    const int B = d.hdr->B, D = d.D;
    const int me = d.hdr->me, mf = d.hdr->mf;
    const double we = me > 0 ? d.hdr->lambda_e / static_cast<double>(me) : 0.0;
    const double wf = mf > 0 ? d.hdr->lambda_f / static_cast<double>(mf) : 0.0;
    for (int s = blockIdx.x; s < B; s += gridDim.x) {
        const int64_t lo = d.atom_ptr[s], hi = d.atom_ptr[s + 1];
        const int ds = d.dsidx[s];
        const bool em = d.emask[s], fm = d.fmask[s];
        const double ws = wf / static_cast<double>(hi - lo);
        double fsum = 0.0;
        for (int64_t a = lo + threadIdx.x; a < hi; a += 128) {
            float* g = d.gF + a * 3 * D;
            for (int q = 0; q < 3 * D; ++q) g[q] = 0.f;
            if (fm) {
                double df[3], sq = 0.0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    df[c] = static_cast<double>(d.F[(a * D + ds) * 3 + c]) - d.Fn[3 * a + c];
                    sq += df[c] * df[c];
                }
                const double dist = sqrt(sq);
                fsum += ws * dist;
                if (dist > 0.0)
#pragma unroll
                    for (int c = 0; c < 3; ++c) g[ds * 3 + c] = static_cast<float>(ws * df[c] / dist);
            }
        }
        red[threadIdx.x] = fsum;
        __syncthreads();
        for (int o = 64; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
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
}

// Fixed-order tree sum of the per-sample terms; the rank's loss goes to the
// header and (as an fp32 hi/lo pair) into the allreduce payload after the grads.
__global__ void __launch_bounds__(1024) k_loss_final(Dev d) {
    __shared__ double re[1024], rf[1024];
    const int B = d.hdr->B;
    double e = 0.0, f = 0.0;
    for (int s = threadIdx.x; s < B; s += 1024) e += d.sample_terms[2 * s], f += d.sample_terms[2 * s + 1];
    re[threadIdx.x] = e, rf[threadIdx.x] = f;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (threadIdx.x < o) re[threadIdx.x] += re[threadIdx.x + o], rf[threadIdx.x] += rf[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double tot = re[0] + rf[0];
        d.hdr->loss_energy = re[0];
        d.hdr->loss_force = rf[0];
        d.hdr->loss_total = tot;
        const float hi = static_cast<float>(tot);
        d.grads[d.NP] = hi;
        d.grads[d.NP + 1] = static_cast<float>(tot - static_cast<double>(hi));
        d.grads[d.NP + 2] = d.hdr->overflow ? 1.f : 0.f;
        d.grads[d.NP + 3] = 1.f;
    }
}

// ------------------------------------------------------ head backward ---
// Scatter-free reverse pass of both heads for one channel per sample (the
// sample's d_s in the train step; a fixed d per pass for a general upstream).
// With s_ij = fcut (gF_i - gF_j).u_ij (u_ji = -u_ij on the symmetric CSR):
//   gT_i = S_i Wa[:,d] + Wb[:,d] (.) W_i,  S_i = sum_j s_ij,  W_i = sum_j s_ij T_j
//   gh_i = We gE_s + gT_i (.) (1 - T_i^2)
// and the per-atom terms Q_i = [T_i (.) W_i / 2 | R_i | S_i] with
// R_ik = sum_j fcut (gF_i.u_ij) rbf_ijk feed dW_fh in k_head_reduce.
template <int H, int K>
__global__ void __launch_bounds__(256) k_head_bwd(Dev d, int pass_ch, int first) {
    constexpr int C = H / 32, QW = H + K + 4;  // row padded to 16 B
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int N = d.hdr->N, L = d.L, D = d.D;
    const float* __restrict__ T = L > 0 ? d.t[L] : d.tanh_emb;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
        const int s = d.sample_of[i];
        const int ch = pass_ch >= 0 ? pass_ch : d.dsidx[s];
        const int irow = L > 0 ? i : __ldg(d.Z + i) - 1;
        const VecF<C> Ti = ldv<C>(T + static_cast<int64_t>(irow) * H + lane * C);
        const float* gfi_p = d.gF + (static_cast<int64_t>(i) * D + ch) * 3;
        const float gfi0 = gfi_p[0], gfi1 = gfi_p[1], gfi2 = gfi_p[2];
        float S = 0.f, Rk = 0.f, W[C];
#pragma unroll
        for (int c = 0; c < C; ++c) W[c] = 0.f;
        const int p0 = d.row_ptr[i], p1 = d.row_ptr[i + 1];
        for (int p = p0; p < p1; ++p) {
            const int j = __ldg(d.col + p);
            const float4 g = __ldg(d.geo + p);
            const float* gfj_p = d.gF + (static_cast<int64_t>(j) * D + ch) * 3;
            const float di = gfi0 * g.x + gfi1 * g.y + gfi2 * g.z;
            const float dj = __ldg(gfj_p) * g.x + __ldg(gfj_p + 1) * g.y + __ldg(gfj_p + 2) * g.z;
            const float sij = g.w * (di - dj);
            const int jrow = L > 0 ? j : __ldg(d.Z + j) - 1;
            const VecF<C> Tj = ldv<C>(T + static_cast<int64_t>(jrow) * H + lane * C);
            S += sij;
#pragma unroll
            for (int c = 0; c < C; ++c) W[c] = fmaf(sij, Tj.v[c], W[c]);
            if (lane < K) Rk = fmaf(g.w * di, __ldg(d.rbf + static_cast<int64_t>(p) * K + lane), Rk);
        }
        float* ghp = d.gh + static_cast<int64_t>(i) * H + lane * C;
        VecF<C> gh;
        if (first) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                float e = 0.f;
                for (int dd = 0; dd < D; ++dd)
                    e = fmaf(d.we[(lane * C + c) * D + dd], d.gE[static_cast<int64_t>(s) * D + dd], e);
                gh.v[c] = e;
            }
        } else {
            gh = ldv<C>(ghp);
        }
        VecF<C> q;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int a = lane * C + c;
            const float gt = S * d.wfh[a * D + ch] + d.wfh[(H + a) * D + ch] * W[c];
            gh.v[c] = fmaf(gt, 1.f - Ti.v[c] * Ti.v[c], gh.v[c]);
            q.v[c] = 0.5f * Ti.v[c] * W[c];
        }
        stv<C>(ghp, gh);
        float* Qi = d.Q + static_cast<int64_t>(i) * QW;
        stv<C>(Qi + lane * C, q);
        if (lane < K) Qi[H + lane] = Rk;
        if (lane == 0) Qi[H + K] = S;
    }
}

// Per-CTA partial dW_fh (all 2H+K rows, channel ch) and dW_e from a
// contiguous atom chunk, summed in atom order with one thread per column.
template <int H, int K>
__global__ void __launch_bounds__(128) k_head_reduce(Dev d, int pass_ch, int first) {
    constexpr int QW = H + K + 4, NQ = 2 * H + K;
    float* acc = dyn_smem<float>();  // [NQ*D] fhead | [H*D] ehead
    const int D = d.D, L = d.L;
    const int W = (NQ + H) * D;
    float* part = d.part_head + static_cast<int64_t>(blockIdx.x) * W;
    for (int e = threadIdx.x; e < W; e += blockDim.x) acc[e] = first ? 0.f : part[e];
    __syncthreads();
    const int N = d.hdr->N;
    const int chunk = (N + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * chunk, i1 = min(N, i0 + chunk);
    const float* __restrict__ T = L > 0 ? d.t[L] : d.tanh_emb;
    const float* __restrict__ hL = L > 0 ? d.h[L] : d.emb;
    for (int i = i0; i < i1; ++i) {
        const int s = d.sample_of[i];
        const int ch = pass_ch >= 0 ? pass_ch : d.dsidx[s];
        const float* Qi = d.Q + static_cast<int64_t>(i) * QW;
        const int irow = L > 0 ? i : d.Z[i] - 1;
        const float S = Qi[H + K];
        for (int q = threadIdx.x; q < NQ; q += blockDim.x) {
            float v;
            if (q < H) v = S * T[static_cast<int64_t>(irow) * H + q];
            else if (q < 2 * H) v = Qi[q - H];
            else v = Qi[H + (q - 2 * H)];
            acc[q * D + ch] += v;
        }
        if (first)
            for (int a = threadIdx.x; a < H; a += blockDim.x) {
                const float hv = hL[static_cast<int64_t>(irow) * H + a];
                for (int dd = 0; dd < D; ++dd) acc[NQ * D + a * D + dd] += hv * d.gE[static_cast<int64_t>(s) * D + dd];
            }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < W; e += blockDim.x) part[e] = acc[e];
}

// ------------------------------------------------------- layer backward ---
// gm = (gh W_u) (.) (1 - mu^2) as a persistent 32-atom tile GEMM, plus the
// per-CTA partial dW_u = sum_i gh_i^T mu_i accumulated in registers across the
// CTA's tiles (16x16 thread grid, (H/16)^2 outputs per thread).
template <int H>
__global__ void __launch_bounds__(256) k_bwd_gemm(Dev d, int l) {
    constexpr int C = H / 32, TM = 32, RPW = TM / 8, RB = H / 16;
    float* sm = dyn_smem<float>();
    float* Wu = sm;             // [H][H] row b, col a
    float* ght = sm + H * H;    // [TM][H]
    float* mut = ght + TM * H;  // [TM][H]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* __restrict__ wu = d.wu[l];
    for (int idx = tid * 4; idx < H * H; idx += blockDim.x * 4)
        *reinterpret_cast<float4*>(Wu + idx) = *reinterpret_cast<const float4*>(wu + idx);
    const int bb = (tid / 16) * RB, aa = (tid % 16) * RB;
    float dW[RB][RB];
#pragma unroll
    for (int x = 0; x < RB; ++x)
#pragma unroll
        for (int y = 0; y < RB; ++y) dW[x][y] = 0.f;
    const int N = d.hdr->N;
    const int ntiles = (N + TM - 1) / TM;
    __syncthreads();
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const int base = ti * TM;
        for (int idx = tid * 4; idx < TM * H; idx += blockDim.x * 4) {
            const int r = idx / H, atom = base + r;
            float4 g = make_float4(0.f, 0.f, 0.f, 0.f), m = g;
            if (atom < N) {
                g = *reinterpret_cast<const float4*>(d.gh + static_cast<int64_t>(atom) * H + idx % H);
                m = *reinterpret_cast<const float4*>(d.mu[l] + static_cast<int64_t>(atom) * H + idx % H);
            }
            *reinterpret_cast<float4*>(ght + idx) = g;
            *reinterpret_cast<float4*>(mut + idx) = m;
        }
        __syncthreads();
        float acc[RPW][C];
#pragma unroll
        for (int r = 0; r < RPW; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[r][c] = 0.f;
        const int r0 = warp * RPW;
#pragma unroll 4
        for (int b = 0; b < H; ++b) {
            const VecF<C> wv = ldv<C>(Wu + b * H + lane * C);
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                const float gv = ght[(r0 + r) * H + b];
#pragma unroll
                for (int c = 0; c < C; ++c) acc[r][c] = fmaf(gv, wv.v[c], acc[r][c]);
            }
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int atom = base + r0 + r;
            if (atom >= N) continue;
            const VecF<C> mv = ldv<C>(mut + (r0 + r) * H + lane * C);
            VecF<C> o;
#pragma unroll
            for (int c = 0; c < C; ++c) o.v[c] = acc[r][c] * (1.f - mv.v[c] * mv.v[c]);
            stv<C>(d.gm + static_cast<int64_t>(atom) * H + lane * C, o);
        }
#pragma unroll 4
        for (int i = 0; i < TM; ++i) {
            float gv[RB], mv[RB];
#pragma unroll
            for (int x = 0; x < RB; ++x) gv[x] = ght[i * H + bb + x], mv[x] = mut[i * H + aa + x];
#pragma unroll
            for (int x = 0; x < RB; ++x)
#pragma unroll
                for (int y = 0; y < RB; ++y) dW[x][y] = fmaf(gv[x], mv[y], dW[x][y]);
        }
        __syncthreads();
    }
    float* part = d.part_wu[l] + static_cast<int64_t>(blockIdx.x) * H * H;
#pragma unroll
    for (int x = 0; x < RB; ++x)
#pragma unroll
        for (int y = 0; y < RB; ++y) part[(bb + x) * H + aa + y] = dW[x][y];
}

// Edge part of layer l's reverse pass, warp per atom, gather form:
//   gt_i = sum_j gm_j (.) filter_ij        (filter symmetric in i, j)
//   dW_f[a,k] += gm_ia t_ja fcut_ij rbf_ijk (per-warp registers, CTA-reduced)
//   gh_i += gt_i (.) (1 - t_i^2)
template <int H, int K>
__global__ void __launch_bounds__(256) k_bwd_edge(Dev d, int l) {
    constexpr int C = H / 32;
    float* red = dyn_smem<float>();  // [warps][H*K]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    float w[C][K], dW[C][K];
    const float* __restrict__ wf = d.wf[l];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int k = 0; k < K; ++k) w[c][k] = wf[(lane * C + c) * K + k], dW[c][k] = 0.f;
    const float* __restrict__ tsrc = l == 0 ? d.tanh_emb : d.t[l];
    const int N = d.hdr->N;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
        const VecF<C> gmi = ldv<C>(d.gm + static_cast<int64_t>(i) * H + lane * C);
        float gt[C];
#pragma unroll
        for (int c = 0; c < C; ++c) gt[c] = 0.f;
        const int p0 = d.row_ptr[i], p1 = d.row_ptr[i + 1];
#pragma unroll 2
        for (int p = p0; p < p1; ++p) {
            const int j = __ldg(d.col + p);
            const float fc = __ldg(&d.geo[p].w);
            float rb[K];
            load_rbf<K>(d.rbf + static_cast<int64_t>(p) * K, rb);
            const VecF<C> gmj = ldv<C>(d.gm + static_cast<int64_t>(j) * H + lane * C);
            const int jrow = l == 0 ? __ldg(d.Z + j) - 1 : j;
            const VecF<C> tj = ldv<C>(tsrc + static_cast<int64_t>(jrow) * H + lane * C);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < K; ++k) acc = fmaf(w[c][k], rb[k], acc);
                gt[c] = fmaf(gmj.v[c], acc * fc, gt[c]);
                const float gg = gmi.v[c] * tj.v[c] * fc;
#pragma unroll
                for (int k = 0; k < K; ++k) dW[c][k] = fmaf(gg, rb[k], dW[c][k]);
            }
        }
        const int irow = l == 0 ? __ldg(d.Z + i) - 1 : i;
        const VecF<C> ti = ldv<C>(tsrc + static_cast<int64_t>(irow) * H + lane * C);
        float* ghp = d.gh + static_cast<int64_t>(i) * H + lane * C;
        VecF<C> gh = ldv<C>(ghp);
#pragma unroll
        for (int c = 0; c < C; ++c) gh.v[c] = fmaf(gt[c], 1.f - ti.v[c] * ti.v[c], gh.v[c]);
        stv<C>(ghp, gh);
    }
    float* mine = red + warp * H * K;
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int k = 0; k < K; ++k) mine[(lane * C + c) * K + k] = dW[c][k];
    __syncthreads();
    const int nwarp = blockDim.x >> 5;
    float* part = d.part_wf[l] + static_cast<int64_t>(blockIdx.x) * H * K;
    for (int e = threadIdx.x; e < H * K; e += blockDim.x) {
        float s = 0.f;
        for (int q = 0; q < nwarp; ++q) s += red[q * H * K + e];
        part[e] = s;
    }
}

// Embedding gradient dE[Z_i - 1] += gh_i, per-CTA partial over a contiguous
// atom chunk, one thread per channel, rows indexed by the batch's Z slots.
template <int H>
__global__ void __launch_bounds__(H) k_embed_grad(Dev d) {
    float* acc = dyn_smem<float>();  // [nslots][H]
    const int ns = d.hdr->nslots;
    for (int e = threadIdx.x; e < ns * H; e += blockDim.x) acc[e] = 0.f;
    __syncthreads();
    const int N = d.hdr->N;
    const int chunk = (N + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * chunk, i1 = min(N, i0 + chunk);
    for (int i = i0; i < i1; ++i) acc[d.zslot[i] * H + threadIdx.x] += d.gh[static_cast<int64_t>(i) * H + threadIdx.x];
    __syncthreads();
    float* part = d.part_emb + static_cast<int64_t>(blockIdx.x) * ns * H;
    for (int e = threadIdx.x; e < ns * H; e += blockDim.x) part[e] = acc[e];
}

// ------------------------------------------------------- grad reduction ---
struct Seg {
    int64_t dst;
    int32_t n, kind;  // kind 0: dense, 1: embedding rows through z_to_slot
    const float* src;
    int32_t ncta, stride;
};
struct SegTable {
    int nseg;
    Seg s[2 * kMaxLayers + 4];
};

// grads[e] = sum over CTAs (index order) of the partials of the tensor that
// owns flat index e (for_each_tensor order).
__global__ void __launch_bounds__(256) k_grad_reduce(Dev d, SegTable tab) {
    const int H = d.H;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int ns = d.hdr->nslots;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < d.NP; e += stride) {
        int q = 0;
        while (q + 1 < tab.nseg && e >= tab.s[q + 1].dst) ++q;
        const Seg& sg = tab.s[q];
        const int64_t off = e - sg.dst;
        float acc = 0.f;
        if (sg.kind == 1) {
            const int zrow = static_cast<int>(off / H), a = static_cast<int>(off % H);
            const int slot = d.z_to_slot[zrow + 1];
            if (slot >= 0)
                for (int c = 0; c < sg.ncta; ++c) acc += sg.src[static_cast<int64_t>(c) * ns * H + slot * H + a];
        } else {
            for (int c = 0; c < sg.ncta; ++c) acc += sg.src[static_cast<int64_t>(c) * sg.stride + off];
        }
        d.grads[e] = acc;
    }
}

// ------------------------------------------------------------ optimizer ---
// Mean over ranks (x 1/G as scale_params does), global norm (fp64, fixed-order
// tree), non-finite check, clip factor; the last CTA finalizes.
__global__ void __launch_bounds__(256) k_opt_norm(Dev d, int G, double inv_g, double clip) {
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
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        d.block_scratch[blockIdx.x] = red[0];
        __threadfence();
        is_last = atomicAdd(&d.hdr->done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last && threadIdx.x == 0) {
        __threadfence();
        double tot = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) tot += d.block_scratch[b];
        const double gn = sqrt(tot);
        double loss = 0.0;
        if (!d.g64_in) loss = (static_cast<double>(d.grads[d.NP]) + static_cast<double>(d.grads[d.NP + 1])) /
                   static_cast<double>(G);
        d.hdr->grad_norm = gn;
        d.hdr->global_loss = loss;
        const bool overflow = !d.g64_in && d.grads[d.NP + 2] > 0.f;
        d.hdr->status = overflow ? 2 : ((!isfinite(loss) || !isfinite(gn)) ? 1 : 0);
        if (d.hdr->status != 0 && !d.g64_in) atomicAdd(d.anomaly, 1u);
        d.hdr->clip_scale = (clip > 0.0 && gn > clip) ? clip / gn : 0.0;
        d.hdr->done_counter = 0;
    }
}

// RmsOptimizer::step with bit-exact fp64 arithmetic given the same gradient;
// refreshes the fp32 working copy and tanh(E) for layer 0's gathers.
__global__ void __launch_bounds__(256) k_opt_step(Dev d, double inv_g, double lr, double decay, double eps) {
    if (d.hdr->status != 0) return;
    const double cs = d.hdr->clip_scale;
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
    }
}

// fp64 master -> fp32 working copy (+ tanh(E)) after a host parameter upload.
__global__ void __launch_bounds__(256) k_params_cast(Dev d) {
    const int64_t emb_n = static_cast<int64_t>(kMaxZ) * d.H;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < d.NP;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float pf = static_cast<float>(d.p64[e]);
        d.p32[e] = pf;
        if (e < emb_n) d.tanh_emb_w[e] = tanhf(pf);
    }
}

}  // namespace lamm_b200
