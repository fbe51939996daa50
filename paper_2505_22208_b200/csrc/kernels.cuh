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
//                     + the per-atom pair counts of S/core.cpp:30-48 (small samples)
//                     + the cell-list binning of large ones
//   k_cell_count .... the pair counts of cell-list, periodic and image samples
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

// Release / acquire fence at GPU scope for the "last block" and grid-barrier
// patterns (writes -> fence -> counter atomic; counter atomic -> fence -> reads):
// acq_rel suffices there, and it is cheaper than __threadfence()'s sequentially
// consistent MEMBAR.SC.GPU.
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

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
// pair_sq: the rounded (dx*dx + dy*dy) + dz*dz that r = sqrt(.) rounds from.
__device__ __forceinline__ double pair_sq(double xi, double yi, double zi, double xj, double yj, double zj,
                                          double& dx, double& dy, double& dz, const double* cell = nullptr) {
    dx = __dsub_rn(xi, xj);
    dy = __dsub_rn(yi, yj);
    dz = __dsub_rn(zi, zj);
    if (cell) min_image(cell, cell + 9, dx, dy, dz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}
__device__ __forceinline__ double pair_dist(double xi, double yi, double zi, double xj, double yj, double zj,
                                            double& dx, double& dy, double& dz, const double* cell = nullptr) {
    return __dsqrt_rn(pair_sq(xi, yi, zi, xj, yj, zj, dx, dy, dz, cell));
}
// The test sqrt_rn(s) < rc without the square root away from the boundary: s below
// rc^2 (1 - 1e-12) is inside and s at or above rc^2 (1 + 1e-12) outside whatever
// the roundings (relative 1e-16 each); only the thin shell between takes the sqrt.
// The decision is the reference's r < cutoff bit for bit.
struct Cut {
    double rc, lo2, hi2;
};
__device__ __forceinline__ Cut make_cut(double rc) { return Cut{rc, rc * rc * (1.0 - 1e-12), rc * rc * (1.0 + 1e-12)}; }
__device__ __forceinline__ bool inside(double s, const Cut& q) {
    return s < q.lo2 || (s < q.hi2 && __dsqrt_rn(s) < q.rc);
}

// The sample's periodic cell in the staged blob ({cell, cinv, m, nimg}), or nullptr.
__device__ __forceinline__ const double* sample_cell(const Dev& d, int s) {
    const StepHeader& hd = *d.hdr;
    if (hd.off_cell == 0) return nullptr;
    const double* c = reinterpret_cast<const double*>(reinterpret_cast<const char*>(d.hdr) + hd.off_cell) +
                      static_cast<int64_t>(kCellDoubles) * s;
    return c[0] != 0.0 ? c + 1 : nullptr;
}

// Candidate images of one sample's pairs: brute-force samples sweep the flattened
// (j, image) index c = j * nimg + img (image order lexicographic in n, the
// reference order i-major / j ascending kept), skipping (i, i, 0). Samples of
// more than kSmallAtoms atoms take the cell lists unless they need images.
struct Images {
    int nimg, w1, w2, m0, m1, m2;
    bool multi;  // flag 2: image shifts / open axes (image_disp), else the minimum image (or none)
};
__device__ __forceinline__ Images sample_images(const double* cell) {
    Images im{1, 1, 1, 0, 0, 0, false};
    if (cell && cell[-1] == 2.0) {
        im.multi = true;
        im.m0 = max(0, static_cast<int>(cell[18])), im.m1 = max(0, static_cast<int>(cell[19]));
        im.m2 = max(0, static_cast<int>(cell[20]));
        im.w1 = 2 * im.m1 + 1, im.w2 = 2 * im.m2 + 1;
        im.nimg = (2 * im.m0 + 1) * im.w1 * im.w2;
    }
    return im;
}
// Who counts a sample's pairs: k_prep's block (small non-periodic samples: the
// reference's molecules), k_cell_count's warp per atom otherwise — over the cell
// lists (large samples without images) or brute force over j (and images).
__device__ __forceinline__ bool counted_in_prep(const double* cell, int n) { return n <= kSmallAtoms && !cell; }
__device__ __forceinline__ bool uses_cells(const double* cell, int n) {
    return n > kSmallAtoms && !(cell && cell[-1] == 2.0);
}
// The images of (i, j) within the cutoff, in image order (n lexicographic), for
// one lane: f(n, dx, dy, dz, sq) is called for each; (i, i, 0) skipped.
template <class F>
__device__ __forceinline__ void for_images(const Images& im, const double* cell, double xi, double yi, double zi,
                                           double xj, double yj, double zj, bool self, const Cut& cut, F&& f) {
    double fr[3];
    image_frac(cell, __dsub_rn(xi, xj), __dsub_rn(yi, yj), __dsub_rn(zi, zj), fr);
    for (int n0 = -im.m0; n0 <= im.m0; ++n0)
        for (int n1 = -im.m1; n1 <= im.m1; ++n1)
            for (int n2 = -im.m2; n2 <= im.m2; ++n2) {
                if (self && n0 == 0 && n1 == 0 && n2 == 0) continue;
                double dx, dy, dz;
                const double sq = image_sq(cell, fr, n0, n1, n2, dx, dy, dz);
                if (inside(sq, cut)) f(dx, dy, dz, sq);
            }
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

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += x;
    }
    return v;
}

// Exclusive scan of src[0, n) into dst (dst may alias src) by one warp, 8
// consecutive values per lane and round so the loads of a round are all in
// flight together; returns the total. src is read through L2 (written by other
// CTAs of this kernel).
__device__ __forceinline__ int warp_excl_scan8(const int32_t* src, int32_t* dst, int n) {
    const int lane = threadIdx.x & 31;
    int run = 0;
    for (int c0 = 0; c0 < n; c0 += 256) {
        int v[8], sum = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = c0 + lane * 8 + u;
            v[u] = k < n ? __ldcg(src + k) : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) sum += v[u];
        const int incl = warp_incl_scan(sum);
        int at = run + incl - sum;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = c0 + lane * 8 + u;
            if (k < n) dst[k] = at;
            at += v[u];
        }
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    return run;
}

// ------------------------------------------------------------ cell lists ---
// Cell of a position in its sample's grid (device.cuh:CellGrid). Binning need not
// be exact — the pair test over the neighbour cells is — only consistent: the
// cell is computed once per atom (k_prep) and stored in acell.
__device__ __forceinline__ int cell_index(const CellGrid& g, const double* cell, double x, double y, double z) {
    int q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double t;
        if (g.periodic) {
            const double* ci = cell + 9;
            t = (x * ci[k] + y * ci[3 + k]) + z * ci[6 + k];
            t = (t - floor(t)) * g.n[k];
        } else {
            t = ((k == 0 ? x : (k == 1 ? y : z)) - g.lo[k]) * g.scale[k];
        }
        q[k] = min(max(static_cast<int>(t), 0), g.n[k] - 1);
    }
    return (q[0] * g.n[1] + q[1]) * g.n[2] + q[2];
}

// Neighbour cell along one axis: c + o (o in -1..1), wrapped when periodic with
// each distinct cell visited once (n = 1: only o = 0; n = 2: o = 0, 1); false
// when the cell does not exist.
__device__ __forceinline__ bool cell_step(const CellGrid& g, int k, int c, int o, int& out) {
    const int n = g.n[k];
    if (g.periodic) {
        if (n == 1 && o != 0) return false;
        if (n == 2 && o < 0) return false;
        out = (c + o + n) % n;
        return true;
    }
    out = c + o;
    return out >= 0 && out < n;
}

// The candidates of one atom as a flat index space: lane q < 27 owns neighbour
// cell q (offsets -1..1 per axis, cell_step's distinct cells only), the warp scan
// of the cell sizes maps candidate t in [0, total) to its slot in the sample's
// cell-ordered atoms, so 32 candidates are tested per round whatever the cell
// occupancy (instead of one round per cell).
struct CellWalk {
    int off, incl, total;
};

__device__ __forceinline__ CellWalk cell_walk_setup(const Dev& d, const CellGrid& g, int c) {
    const int lane = threadIdx.x & 31;
    const int c2 = c % g.n[2], c1 = (c / g.n[2]) % g.n[1], c0 = c / (g.n[1] * g.n[2]);
    int b = 0, n = 0, x0, x1, x2;
    if (lane < 27 && cell_step(g, 0, c0, lane / 9 - 1, x0) && cell_step(g, 1, c1, (lane / 3) % 3 - 1, x1) &&
        cell_step(g, 2, c2, lane % 3 - 1, x2)) {
        const int q = (x0 * g.n[1] + x1) * g.n[2] + x2;
        b = __ldg(d.cstart + g.base + q);
        n = __ldg(d.cstart + g.base + q + 1) - b;
    }
    CellWalk w;
    w.incl = warp_incl_scan(n);
    w.off = b - (w.incl - n);
    w.total = __shfl_sync(0xffffffffu, w.incl, 31);
    return w;
}

// Slot (in the sample's cpos) of candidate t < total; every lane must call it.
__device__ __forceinline__ int cell_walk_slot(const CellWalk& w, int t) {
    int q = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
        if (t >= __shfl_sync(0xffffffffu, w.incl, q + step - 1)) q += step;
    return t + __shfl_sync(0xffffffffu, w.off, q);
}

// Block-wide (128 threads): the grid of sample s (bounding box or lattice), each
// atom's cell, a counting sort of the atoms by cell into cpos, and the cell
// offsets. lptr holds the atom's rank inside its cell until k_cell_count
// overwrites it with the row offset.
// mn / mx: this thread's bounding box of the atoms it positioned (k_prep's loop).
__device__ void bin_sample(const Dev& d, int s, int64_t lo, int64_t hi, const double* cell, double (&mn)[3],
                           double (&mx)[3]) {
    __shared__ double red[4][6];
    __shared__ CellGrid sg;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = fmin(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < 3; ++k) red[w][k] = mn[k], red[w][3 + k] = mx[k];
    __syncthreads();
    if (tid == 0) {
        CellGrid g{};
        const double s0 = d.rc * (1.0 + 1e-9);  // slack far above the binning's rounding
        double amax = 0.0;
        for (int k = 0; k < 3; ++k) {
            for (int q = 1; q < 4; ++q) red[0][k] = fmin(red[0][k], red[q][k]), red[0][3 + k] = fmax(red[0][3 + k], red[q][3 + k]);
            amax = fmax(amax, fmax(fabs(red[0][k]), fabs(red[0][3 + k])));
        }
        g.periodic = cell != nullptr;
        bool ok = true;
        for (int k = 0; k < 3; ++k) {
            double cells;
            if (g.periodic) {  // slab width along lattice direction k = 1 / |column k of cell^-1|
                const double* ci = cell + 9;
                const double b = sqrt(ci[k] * ci[k] + ci[3 + k] * ci[3 + k] + ci[6 + k] * ci[6 + k]);
                cells = floor(1.0 / (b * s0));
                ok &= amax * b < 1e3;  // fractional coordinates small enough to bin accurately
            } else {
                const double ext = red[0][3 + k] - red[0][k];
                cells = floor(ext / s0);
                ok &= ext < 1e7;
                g.lo[k] = red[0][k];
                g.scale[k] = cells >= 1.0 ? fmin(cells, 1024.0) / ext : 0.0;
            }
            g.n[k] = static_cast<int>(fmax(1.0, fmin(cells, 1024.0)));
        }
        if (!ok) g.n[0] = g.n[1] = g.n[2] = 1;  // degenerate input: one cell = brute force
        // at most 4 cells per atom (+64): halve the finest axis (wider cells stay valid)
        const int64_t cap = 4 * (hi - lo) + 64;
        while (static_cast<int64_t>(g.n[0]) * g.n[1] * g.n[2] > cap) {
            const int k = g.n[0] >= g.n[1] && g.n[0] >= g.n[2] ? 0 : (g.n[1] >= g.n[2] ? 1 : 2);
            const int n2 = max(1, g.n[k] / 2);
            if (!g.periodic && g.scale[k] != 0.0) g.scale[k] *= static_cast<double>(n2) / g.n[k];
            g.n[k] = n2;
        }
        g.base = static_cast<int>(4 * lo + 65 * static_cast<int64_t>(s));
        sg = g;
        d.cgrid[s] = g;
        d.sdone[s] = 0u;
    }
    __syncthreads();
    const CellGrid g = sg;
    const int ncell = g.n[0] * g.n[1] * g.n[2];
    int32_t* cs = d.cstart + g.base;
    for (int q = tid; q <= ncell; q += blockDim.x) cs[q] = 0;
    __syncthreads();
    for (int64_t a0 = lo + tid; a0 < hi; a0 += 4 * blockDim.x) {
        int c[4], r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t a = a0 + u * blockDim.x;
            if (a < hi) c[u] = cell_index(g, cell, d.x[a], d.y[a], d.z[a]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (a0 + u * blockDim.x < hi) r[u] = atomicAdd(cs + c[u], 1);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t a = a0 + u * blockDim.x;
            if (a < hi) d.acell[a] = c[u], d.lptr[a] = r[u];
        }
    }
    __syncthreads();
    __shared__ int scratch[4];
    int run = 0;
    for (int q0 = 0; q0 < ncell; q0 += blockDim.x) {
        const int q = q0 + tid;
        const int v = q < ncell ? __ldcg(cs + q) : 0;
        int tot;
        const int ex = block_excl_scan128(v, scratch, &tot);
        if (q < ncell) cs[q] = run + ex;
        run += tot;
    }
    if (tid == 0) cs[ncell] = run;
    __syncthreads();
    for (int64_t a0 = lo + tid; a0 < hi; a0 += 4 * blockDim.x) {
        int at[4];
        double4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t a = a0 + u * blockDim.x;
            if (a < hi) at[u] = d.acell[a], v[u] = make_double4(d.x[a], d.y[a], d.z[a], __longlong_as_double(a));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (a0 + u * blockDim.x < hi) at[u] = __ldcg(cs + at[u]) + d.lptr[a0 + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (a0 + u * blockDim.x < hi) d.cpos[lo + at[u]] = v[u];
    }
}

// The sample offsets (scan of the per-sample pair totals), P, the capacity flag,
// row_ptr[N], the partition defaults and the CSR padding; one warp, after every
// sample's total is final (the last block of k_prep, or the last sample of
// k_cell_count when the batch has cell-list samples).
__device__ void finalize_csr_warp(const Dev& d, int Q) {
    const int lane = threadIdx.x & 31;
    const int B = d.hdr->B, N = d.hdr->N;
    const int run = warp_excl_scan8(d.stot, d.soff, B);
    const bool over = static_cast<int64_t>(run) > d.Pcap;
    if (lane == 0) {
        d.hdr->P = run;
        d.hdr->overflow = over ? 1 : 0;
        d.row_ptr[N] = run;
    }
    // partitions: cut by k_nbr_fill when there are edges; all empty on overflow
    // (the step is discarded and rerun with more capacity); no edges: the last
    // partition walks every atom (edge-less begin/end)
    if (over || run == 0)
        for (int q = lane; q < Q; q += 32) d.part_lo[q] = 0;
    if (lane == 0) d.part_lo[Q] = over ? 0 : N;
    if (!over)  // CSR padding read by the edge kernels' block staging: valid source atom 0
        for (int x = lane; x < kChunk + 8; x += 32) d.col[run + x] = 0, d.colz[run + x] = 0, d.dst[run + x] = N;
}


// Also the CSR row offsets (S/core.cpp:30-48 order: i-major): each sample's
// block scans its atoms' pair counts (lptr = offset inside the sample, stot =
// sample total); the last block to finish scans the sample totals (soff), sets
// P / the capacity-overflow flag / row_ptr[N] / the CSR padding, so the
// neighbour fill can place every atom's row without a separate scan kernel.
// Q: edge-kernel partitions (k_nbr_fill cuts them while writing row_ptr).
__global__ void __launch_bounds__(128, 4) k_prep(Dev d, BatchArrays out, int Q) {
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
    __shared__ double stage[4][128];
    __shared__ double sp[3][kSmallAtoms];  // positions of a small sample
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
        }
        // S/denoise.cpp:14-19 (sequential sum, then (1/n) * sum) and S/loss.cpp:117-121
        // (sequential sum of the reference energies): the per-atom terms are staged
        // 128 at a time in shared memory and thread 0 adds them in index order
        const bool need_mean = is_dn && d.denoise_scheme, need_tab = d.use_table && em[s];
        double m0 = 0.0, m1 = 0.0, m2 = 0.0, total = 0.0;
        if (need_mean || need_tab) {
            for (int64_t c0 = lo; c0 < hi; c0 += 128) {
                const int64_t a = c0 + threadIdx.x;
                if (a < hi) {
                    if (need_mean)
                        stage[0][threadIdx.x] = noise[3 * a], stage[1][threadIdx.x] = noise[3 * a + 1],
                        stage[2][threadIdx.x] = noise[3 * a + 2];
                    if (need_tab) {  // absent element: -0.0 leaves the sum unchanged, as the skip does
                        const int z = Z[a];
                        stage[3][threadIdx.x] = d.rho_has[dsi * 119 + z] ? d.rho[dsi * 119 + z] : -0.0;
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    const int n = static_cast<int>(hi - c0 < 128 ? hi - c0 : 128);
                    if (need_mean)
                        for (int k = 0; k < n; ++k)
                            m0 = __dadd_rn(m0, stage[0][k]), m1 = __dadd_rn(m1, stage[1][k]), m2 = __dadd_rn(m2, stage[2][k]);
                    if (need_tab)
                        for (int k = 0; k < n; ++k) total = __dadd_rn(total, stage[3][k]);
                }
                __syncthreads();
            }
        }
        if (threadIdx.x == 0) {
            if (need_mean) {
                const double sc = __ddiv_rn(1.0, static_cast<double>(hi - lo));
                m0 = __dmul_rn(sc, m0), m1 = __dmul_rn(sc, m1), m2 = __dmul_rn(sc, m2);
            }
            mean[0] = m0, mean[1] = m1, mean[2] = m2;
            double e = E[s];
            if (need_tab) e = __ddiv_rn(__dsub_rn(__dsub_rn(e, total), d.tmean[dsi]), d.tstd[dsi]);
            d.En[s] = e;
        }
        __syncthreads();
        const double fs = d.use_table ? __ddiv_rn(1.0, d.tfstd[dsi]) : 1.0;
        // the Eq. (5) weight of the atom's force term (S/loss.cpp:186-212): lambda_F / (sum m_F * n)
        const int mfs = hd.mf;
        const double fwa = fm[s] && mfs > 0 ? hd.lambda_f / (static_cast<double>(mfs) * static_cast<double>(hi - lo)) : 0.0;
        double bmn[3] = {INFINITY, INFINITY, INFINITY}, bmx[3] = {-INFINITY, -INFINITY, -INFINITY};  // bounding box
        // 4 atoms per thread and round, every load issued before the first store
        // (large samples are latency-bound here: one block walks all their atoms)
        for (int64_t a0 = lo + threadIdx.x; a0 < hi; a0 += 4 * blockDim.x) {
            double pin[4][3], src[4][3];
            int zz[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t a = a0 + u * blockDim.x;
                if (a < hi) {
                    zz[u] = Z[a];
#pragma unroll
                    for (int c = 0; c < 3; ++c) pin[u][c] = pos[3 * a + c], src[u][c] = is_dn ? noise[3 * a + c] : F[3 * a + c];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t a = a0 + u * blockDim.x;
                if (a >= hi) break;
                d.sample_of[a] = s;
                d.chan[a] = dsi;
                d.fw[a] = fwa;
                out.Z[a] = zz[u];
                out.zslot[a] = z2s[zz[u]];
                double xyz[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double lab;
                    if (is_dn) {
                        const double eff = d.denoise_scheme ? __dsub_rn(src[u][c], mean[c]) : src[u][c];
                        xyz[c] = __dadd_rn(pin[u][c], eff);
                        lab = __dmul_rn(-1.0, eff);
                    } else {
                        xyz[c] = pin[u][c];
                        lab = src[u][c];
                    }
                    d.Fn[3 * a + c] = d.use_table ? __dmul_rn(fs, lab) : lab;
                }
                d.x[a] = xyz[0], d.y[a] = xyz[1], d.z[a] = xyz[2];
#pragma unroll
                for (int k = 0; k < 3; ++k) bmn[k] = fmin(bmn[k], xyz[k]), bmx[k] = fmax(bmx[k], xyz[k]);
                if (hi - lo <= kSmallAtoms)  // the pair counts below read them from shared memory
                    sp[0][a - lo] = xyz[0], sp[1][a - lo] = xyz[1], sp[2][a - lo] = xyz[2];
            }
        }
        __syncthreads();
        const double* cell = sample_cell(d, s);
        const int n = static_cast<int>(hi - lo);
        if (!counted_in_prep(cell, n)) {  // counted by k_cell_count (warp per atom)
            if (uses_cells(cell, n)) {
                bin_sample(d, s, lo, hi, cell, bmn, bmx);
                __syncthreads();
            } else if (threadIdx.x == 0) {
                d.sdone[s] = 0u;
            }
            continue;
        }
        // neighbour counts of the sample (S/core.cpp:30-48), warp per atom, from the
        // positions this block just staged in shared memory (visible after the barrier)
        const int lane = threadIdx.x & 31;
        const Cut cut = make_cut(d.rc);
        for (int il = threadIdx.x >> 5; il < n; il += blockDim.x >> 5) {
            const double xi = sp[0][il], yi = sp[1][il], zi = sp[2][il];
            int cnt = 0;
            for (int j0 = 0; j0 < n; j0 += 32) {
                const int jl = j0 + lane;
                bool in = false;
                if (jl < n && jl != il) {
                    double dx, dy, dz;
                    in = inside(pair_sq(xi, yi, zi, sp[0][jl], sp[1][jl], sp[2][jl], dx, dy, dz, cell), cut);
                }
                cnt += __popc(__ballot_sync(0xffffffffu, in));
            }
            if (lane == 0) d.cnt[lo + il] = cnt;
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
    // the last block: offsets of the samples, P, overflow, row_ptr[N], padding —
    // unless cell-list samples are still to be counted (k_cell_count does it then)
    fence_gpu();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&d.hdr->done_counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    fence_gpu();
    if (hd.n_large == 0 && threadIdx.x < 32) finalize_csr_warp(d, Q);
    if (threadIdx.x == 0) d.hdr->done_counter = 0;
}

// Pair counts of the atoms of cell-list samples (kSmallAtoms < n) and periodic
// samples: the exact test of k_prep's sweep against the atoms of the 27 neighbour
// cells (or every j and its images). Each warp takes a contiguous run of atoms, so
// its atoms share their sample (per-sample data loaded once, one completion
// atomic per run instead of one fenced atomic per atom) and mostly their neighbour
// cells (L1). The warp that completes a sample scans the sample's row offsets;
// the one that finishes the last such sample runs finalize_csr_warp.
__global__ void __launch_bounds__(256, 2) k_cell_count(Dev d, int Q) {
    constexpr int kR = 4;  // candidate rounds (32 candidates each) whose loads are in flight together
    __shared__ uint32_t wbits[8][kMaskWords];
    pdl_enter();
    const StepHeader& hd = *d.hdr;
    const int n_large = hd.n_large;
    if (n_large == 0) return;
    const int N = hd.N;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int per = (N + nw - 1) / nw;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int i1 = min(N, (wid + 1) * per);
    const Cut cut = make_cut(d.rc);
    int i = min(N, wid * per);
    while (i < i1) {
        const int s = d.sample_of[i];
        const int lo = static_cast<int>(d.atom_ptr[s]), hi = static_cast<int>(d.atom_ptr[s + 1]);
        const int iend = min(i1, hi);  // this warp's run of sample s
        const double* cell = sample_cell(d, s);
        if (counted_in_prep(cell, hi - lo)) {
            i = iend;
            continue;
        }
        const Images im = sample_images(cell);
        const bool cells = !im.multi && uses_cells(cell, hi - lo);
        // samples of <= kMaskAtoms atoms: the hits as a bitmask over the sample's
        // atoms, kept for the fill (no second pass of pair tests)
        const bool keep = cells && hi - lo <= kMaskAtoms;
        uint32_t* bits = wbits[threadIdx.x >> 5];
        const int nrun = iend - i;
        for (; i < iend; ++i) {
            const double xi = d.x[i], yi = d.y[i], zi = d.z[i];
            int cnt = 0;
            if (im.multi) {  // image sample: lane per source atom j, its images in a loop
                int own = 0;
                for (int j = lo + lane; j < hi; j += 32)
                    for_images(im, cell, xi, yi, zi, d.x[j], d.y[j], d.z[j], j == i, cut,
                               [&](double, double, double, double) { ++own; });
                cnt = __reduce_add_sync(0xffffffffu, own);
            } else if (!cells) {  // small periodic sample: minimum image, lane per j
                int own = 0;
                for (int j = lo + lane; j < hi; j += 32) {
                    double dx, dy, dz;
                    own += (j != i && inside(pair_sq(xi, yi, zi, d.x[j], d.y[j], d.z[j], dx, dy, dz, cell), cut)) ? 1 : 0;
                }
                cnt = __reduce_add_sync(0xffffffffu, own);
            } else {
                if (keep) {
#pragma unroll
                    for (int q = 0; q < kMaskWords / 32; ++q) bits[32 * q + lane] = 0u;
                    __syncwarp();
                }
                const CellWalk w = cell_walk_setup(d, d.cgrid[s], d.acell[i]);
                for (int t0 = 0; t0 < w.total; t0 += 32 * kR) {
                    double4 p[kR];
#pragma unroll
                    for (int u = 0; u < kR; ++u) {  // every lane runs the slot search (shuffles)
                        const int t = t0 + 32 * u + lane;
                        const int k = cell_walk_slot(w, t);
                        if (t < w.total) p[u] = d.cpos[lo + k];
                    }
#pragma unroll
                    for (int u = 0; u < kR; ++u) {
                        bool in = false;
                        int j = 0;
                        if (t0 + 32 * u + lane < w.total) {
                            double dx, dy, dz;
                            j = static_cast<int>(__double_as_longlong(p[u].w));
                            in = j != i && inside(pair_sq(xi, yi, zi, p[u].x, p[u].y, p[u].z, dx, dy, dz, cell), cut);
                        }
                        if (keep && in) atomicOr(bits + ((j - lo) >> 5), 1u << ((j - lo) & 31));
                        cnt += __popc(__ballot_sync(0xffffffffu, in));
                    }
                }
                if (keep) {
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < kMaskWords / 32; ++q)
                        d.cmask[static_cast<int64_t>(i) * kMaskWords + 32 * q + lane] = bits[32 * q + lane];
                    __syncwarp();
                }
            }
            if (lane == 0) d.cnt[i] = cnt;
        }
        unsigned last = 0;
        if (lane == 0) {
            fence_gpu();  // the run's counts before its completion
            last = atomicAdd(d.sdone + s, static_cast<unsigned>(nrun)) + nrun == static_cast<unsigned>(hi - lo);
        }
        if (!__shfl_sync(0xffffffffu, last, 0)) continue;
        fence_gpu();
        const int run = warp_excl_scan8(d.cnt + lo, d.lptr + lo, hi - lo);  // the sample's row offsets
        unsigned glast = 0;
        if (lane == 0) {
            d.stot[s] = run;
            fence_gpu();
            glast = atomicAdd(&d.hdr->large_done, 1u) == static_cast<unsigned>(n_large - 1);
        }
        if (!__shfl_sync(0xffffffffu, glast, 0)) continue;
        fence_gpu();
        finalize_csr_warp(d, Q);
        if (lane == 0) d.hdr->large_done = 0;
    }
}

// Edge geometry of pair p = (i, j) from its fp64 difference and distance: unit
// (1/r)*d (S/core.cpp:43), fcut (S/model.cpp:17) and the Gaussians (S/model.cpp:20-27)
// in the three layouts the edge kernels read.
template <int K>
__device__ __forceinline__ void emit_pair(const Dev& d, int p, int i, int j, double r, double dx, double dy, double dz,
                                          float wf, float invf, float rc_inv) {
    d.col[p] = j;
    d.colz[p] = d.Z[j] - 1;
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

// Warp per atom i, writing row i of the CSR (i-major, j ascending). Small samples:
// the same sweep as the count in k_prep, lanes that hold a neighbour compact into
// the row with popc(ballot & lanes_below). Cell-list samples: per window of 1024
// consecutive j, the exact test over the neighbour cells sets bit j of a per-warp
// shared-memory mask, the set bits are listed in ascending j (one mask word per
// lane, warp scan of the popcounts) and the lanes emit the listed pairs.
// The edge walks cost ~0.1 us per edge and ~0.4-0.5 us per destination atom (its
// segment flush and per-atom loads) per group (%globaltimer fit on the layer
// backward at cfg2): a 4-edge weight per atom in the partition cut. Measured: cfg2
// step -0.6 %, the 28-edges-per-atom supercell batch +0.8 % (profiles/README.md).
constexpr int kAtomCost = 4;

template <int K>
__global__ void __launch_bounds__(256, 4) k_nbr_fill(Dev d, int Q) {
    constexpr int kWin = 1024;
    __shared__ uint32_t wbits[8][kWin / 32];
    __shared__ int wlist[8][kWin];
    pdl_enter();
    if (d.hdr->overflow) return;
    const int N = d.hdr->N;
    const int64_t P = d.hdr->P;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const double width = d.rc / static_cast<double>(K - 1);
    const float wf = static_cast<float>(width), invf = static_cast<float>(1.0 / (2.0 * width * width));
    const float rc_inv = static_cast<float>(1.0 / d.rc);
    const Cut cut = make_cut(d.rc);
    if (blockIdx.x == 0)  // the CSR padding's geometry: finite zeros (masked edges must not carry stale NaN)
        for (int x = threadIdx.x; x < (kChunk + 8) * K; x += blockDim.x) {
            const int64_t p = P + x / K;
            const int k = x % K;
            if (k == 0) d.geo[p] = make_float4(0.f, 0.f, 0.f, 0.f);
            d.rbf[rbf_idx<K>(p, k)] = 0.f;
            d.rbfl[rbf_idx<K>(p, k)] = 0.f;
            d.rbfp[p * K + k] = 0.f;
        }
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
            // edge-kernel partitions balanced on the walk's cost, kAtomCost edges' worth per
            // atom (its begin / end) plus one per edge: with x_i = row_ptr[i] + kAtomCost i
            // and T = P + kAtomCost N, part_lo[q] = first atom with x_i >= floor(T q / Q)
            if (P > 0) {
                const int64_t T = P + static_cast<int64_t>(kAtomCost) * N;
                const int64_t x = static_cast<int64_t>(base) + static_cast<int64_t>(kAtomCost) * i;
                const int64_t xprev = i == 0 ? -1 : x - d.cnt[i - 1] - kAtomCost;  // x_{i-1}
                const int64_t qlo = i == 0 ? 0 : ((xprev + 1) * Q + T - 1) / T;
                int64_t qhi = ((x + 1) * Q + T - 1) / T - 1;
                if (qhi > Q - 1) qhi = Q - 1;
                for (int64_t q = qlo; q <= qhi; ++q) d.part_lo[q] = i;
                if (i == N - 1)  // targets in (x_{N-1}, T] start at atom N
                    for (int64_t q = ((x + 1) * Q + T - 1) / T; q < Q; ++q) d.part_lo[q] = N;
            }
        }
        const Images im = sample_images(cell);
        if (im.multi) {  // image sample: lane per source atom j (ascending), its hits in image order
            for (int j0 = lo; j0 < hi; j0 += 32) {
                const int j = j0 + lane;
                int own = 0;
                if (j < hi)
                    for_images(im, cell, xi, yi, zi, d.x[j], d.y[j], d.z[j], j == i, cut,
                               [&](double, double, double, double) { ++own; });
                const int incl = warp_incl_scan(own);
                int at = base + incl - own;
                if (j < hi)
                    for_images(im, cell, xi, yi, zi, d.x[j], d.y[j], d.z[j], j == i, cut,
                               [&](double dx, double dy, double dz, double sq) {
                                   emit_pair<K>(d, at++, i, j, __dsqrt_rn(sq), dx, dy, dz, wf, invf, rc_inv);
                               });
                base += __shfl_sync(0xffffffffu, incl, 31);
            }
            continue;
        }
        if (!uses_cells(cell, hi - lo)) {
            for (int j0 = lo; j0 < hi; j0 += 32) {
                const int j = j0 + lane;
                bool in = false;
                double dx = 0, dy = 0, dz = 0, r = 0;
                if (j < hi && j != i) {
                    r = pair_dist(xi, yi, zi, d.x[j], d.y[j], d.z[j], dx, dy, dz, cell);
                    in = r < d.rc;
                }
                const unsigned mask = __ballot_sync(0xffffffffu, in);
                if (in) emit_pair<K>(d, base + __popc(mask & ((1u << lane) - 1u)), i, j, r, dx, dy, dz, wf, invf, rc_inv);
                base += __popc(mask);
            }
            continue;
        }
        const CellGrid g = d.cgrid[s];
        const bool kept = hi - lo <= kMaskAtoms;  // k_cell_count left the row's bitmask
        const CellWalk cw = kept ? CellWalk{} : cell_walk_setup(d, g, d.acell[i]);
        uint32_t* bits = wbits[wib];
        int* list = wlist[wib];
        for (int w0 = lo; w0 < hi; w0 += kWin) {
            bits[lane] = kept ? __ldcg(d.cmask + static_cast<int64_t>(i) * kMaskWords + (w0 - lo) / 32 + lane) : 0u;
            __syncwarp();
            for (int t0 = 0; !kept && t0 < cw.total; t0 += 32) {
                const int k = cell_walk_slot(cw, t0 + lane);
                if (t0 + lane < cw.total) {
                    const double4 p = d.cpos[lo + k];
                    const int j = static_cast<int>(__double_as_longlong(p.w));
                    double dx, dy, dz;
                    if (j >= w0 && j < w0 + kWin && j != i && inside(pair_sq(xi, yi, zi, p.x, p.y, p.z, dx, dy, dz, cell), cut))
                        atomicOr(bits + ((j - w0) >> 5), 1u << ((j - w0) & 31));
                }
            }
            __syncwarp();
            uint32_t word = bits[lane];
            const int c = __popc(word);
            const int incl = warp_incl_scan(c);
            int at = incl - c;
            while (word) {
                list[at++] = w0 + 32 * lane + __ffs(word) - 1;
                word &= word - 1u;
            }
            __syncwarp();
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            for (int k = lane; k < total; k += 32) {
                const int j = list[k];
                double dx, dy, dz;
                const double r = pair_dist(xi, yi, zi, d.x[j], d.y[j], d.z[j], dx, dy, dz, cell);
                emit_pair<K>(d, base + k, i, j, r, dx, dy, dz, wf, invf, rc_inv);
            }
            base += total;
            __syncwarp();
        }
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
    if (with_energy == 2 && !d.hdr->overflow) {  // train step: the head backward's per-edge scalars
        const int P = d.hdr->P;                     // (S/model.cpp:318-340); on overflow P > capacity
        for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
            const int i = d.dst[p], j = d.col[p];
            const float4 gv = d.geo[p];
            const float4 gi = d.gFc[i], gj = d.gFc[j];
            const float di = gi.x * gv.x + gi.y * gv.y + gi.z * gv.z;
            const float dj = gj.x * gv.x + gj.y * gv.y + gj.z * gv.z;
            d.sij[p] = make_float2(gv.w * (di - dj), di);
        }
    }
    double* ered = dyn_smem<double>();  // [D][128] when with_energy
    __shared__ double red[128], red2[128];
    __shared__ bool last;
    const int B = d.hdr->B, D = d.D;
    const int me = d.hdr->me, mf = d.hdr->mf;
    const double we = me > 0 ? d.hdr->lambda_e / static_cast<double>(me) : 0.0;
    const double wf = mf > 0 ? d.hdr->lambda_f / static_cast<double>(mf) : 0.0;
    for (int s = blockIdx.x; s < B; s += gridDim.x) {
        const int ds = d.dsidx[s];
        const int64_t lo = d.atom_ptr[s], hi = d.atom_ptr[s + 1];
        const bool em = d.emask[s], fm = d.fmask[s];
        if (with_energy == 2) {  // train step: per-atom terms from k_force_out, summed in a fixed order
            double es = 0.0, fs = 0.0;
            for (int64_t a = lo + threadIdx.x; a < hi; a += 128) es += d.eatom[a], fs += d.fterm[a];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                es += __shfl_xor_sync(0xffffffffu, es, o), fs += __shfl_xor_sync(0xffffffffu, fs, o);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = es, red2[threadIdx.x >> 5] = fs;
            __syncthreads();
            if (threadIdx.x == 0) {
                const double E = ((red[0] + red[1]) + red[2]) + red[3];
                d.Epred[static_cast<int64_t>(s) * D + ds] = E;
                red[0] = ((red2[0] + red2[1]) + red2[2]) + red2[3];
                double et = 0.0;
                if (em) et = we * fabs(E - d.En[s]);
                d.sample_terms[2 * s] = et;
                d.sample_terms[2 * s + 1] = fm ? red[0] : 0.0;
            }
            __syncthreads();
            if (threadIdx.x < D) {
                float ge = 0.f;
                if (threadIdx.x == ds && em) {
                    const double diff = d.Epred[static_cast<int64_t>(s) * D + ds] - d.En[s];
                    ge = diff > 0.0 ? static_cast<float>(we) : (diff < 0.0 ? static_cast<float>(-we) : 0.f);
                }
                d.gE[static_cast<int64_t>(s) * D + threadIdx.x] = ge;
            }
            __syncthreads();
            continue;
        }
        if (with_energy) sample_energy_own(d, s, ds, ered);
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
        fence_gpu();
        last = atomicAdd(&d.hdr->done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    fence_gpu();
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
        fence_gpu();
        last = atomicAdd(&d.hdr->done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    fence_gpu();
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
            int c0 = g, cs = 8, ncta = sg.ncta;
            int64_t stride = sg.stride;
            if (sg.kind == 1) {
                const int zrow = static_cast<int>(off / H), a = static_cast<int>(off % H);
                const int slot = d.z_to_slot[zrow + 1];
                if (slot >= 0) base = sg.src + slot * H + a;
                stride = static_cast<int64_t>(ns) * H;
            } else if (sg.kind == 2) {
                // column-split partials: CTA c holds columns [np*nc, np*nc+nc), np = c % (H/nc);
                // only the CTAs that had a 128-atom tile wrote one (c < ntiles)
                const int nc = sg.stride / H, nsplit = H / nc;
                const int b = static_cast<int>(off / H), a = static_cast<int>(off % H), np = a / nc;
                base = sg.src + b * nc + (a - np * nc);
                c0 = np + nsplit * g;
                cs = 8 * nsplit;
                ncta = min(ncta, (d.hdr->N + 127) / 128 * nsplit);
            } else {
                base = sg.src + off;
            }
            if (base) {  // 8 loads in flight per step, summed in stream order
                int c = c0;
                for (; c + 7 * cs < ncta; c += 8 * cs) {
                    float v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = __ldcg(base + (c + u * cs) * stride);
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc += v[u];
                }
                for (; c < ncta; c += cs) acc += __ldcg(base + c * stride);
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
        fence_gpu();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            fence_gpu();
            atomicAdd(gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(64);
        }
        fence_gpu();
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
    // a step submitted behind a failed (overflow / non-finite) in-flight step is
    // skipped (status 3) so the host can rerun the chain in order
    const bool chain = d.hdr->chain != 0;
    const bool poisoned = chain && *reinterpret_cast<volatile unsigned int*>(d.anomaly + 8) != 0u;
    const int status = overflow ? 2 : ((!isfinite(loss) || !isfinite(gn)) ? 1 : (poisoned ? 3 : 0));
    const double cs = (clip > 0.0 && gn > clip) ? clip / gn : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        d.hdr->grad_norm = gn;
        d.hdr->global_loss = loss;
        d.hdr->status = status;
        d.hdr->clip_scale = cs;
        if ((status == 1 || status == 2) && !d.g64_in) atomicAdd(d.anomaly, 1u);
        if ((status == 1 || status == 2) && chain) d.anomaly[8] = 1u;
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
