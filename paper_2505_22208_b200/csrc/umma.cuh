// umma.cuh - minimal tcgen05 (5th-gen tensor core) + TMEM toolkit for sm_100a,
// written against the PTX ISA: shared-memory matrix descriptors, the kind::tf32
// instruction descriptor, MMA issue/commit, TMEM alloc and loads.
//
// Operand layout used throughout: K-major, no swizzle ("interleaved") canonical
// tiles of fp32/tf32. A core matrix is 8 rows x 16 bytes (4 elements) stored
// contiguously (128 B); core matrices adjacent in K are 128 B apart (LBO) and
// 8-row groups are (KW/4)*128 B apart (SBO) for a tile KW elements wide. One
// kind::tf32 MMA consumes K = 8 (two core matrices), so K-step s starts s*256 B
// into the tile.
//
// fp32 accuracy from tf32 tensor cores: every operand x is split
// x = hi + lo with hi = tf32(x) (round-to-nearest) and lo = x - hi (exact in
// fp32, its tf32 truncation keeps ~22 significant bits of x in total), and each
// product is accumulated as hi*hi + hi*lo + lo*hi ("3xTF32"): ~1e-7 relative,
// well inside the 1e-4 parity bar, at one third of the tf32 tensor rate.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lamm_b200 {
namespace umma {

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// Element (row m, col k) of a [rows][KW] K-major canonical fp32 tile.
__device__ __forceinline__ int kidx(int m, int k, int KW) {
    return (((m >> 3) * (KW >> 2) + (k >> 2)) << 5) + ((m & 7) << 2) + (k & 3);
}

// SM100 shared-memory matrix descriptor, SWIZZLE_NONE, version 1.
__device__ __forceinline__ uint64_t sdesc(const void* tile, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr(tile) >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm100)
    return d;                              // base offset 0, layout SWIZZLE_NONE (bits 61-63 = 0)
}

// Descriptor of K-step s of a K-major canonical tile KW elements wide.
__device__ __forceinline__ uint64_t kdesc(const float* tile, int s, int KW) {
    return sdesc(tile + s * 64, 128u, static_cast<uint32_t>((KW >> 2) * 128));
}

// kind::tf32 instruction descriptor: D fp32, A/B tf32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// 3xTF32 product accumulation for one K-step: D (+)= Ahi Bhi + Ahi Blo + Alo Bhi.
__device__ __forceinline__ void mma3(uint32_t tmem_d, uint64_t ahi, uint64_t alo, uint64_t bhi, uint64_t blo,
                                     uint32_t idesc, uint32_t acc) {
    mma_tf32(tmem_d, ahi, bhi, idesc, acc);
    mma_tf32(tmem_d, ahi, blo, idesc, 1u);
    mma_tf32(tmem_d, alo, bhi, idesc, 1u);
}

// Arrives on an mbarrier when all previously issued MMAs of this thread finish.
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
                 : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// Generic-proxy shared-memory writes -> visible to the tensor core (async proxy).
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Whole-warp TMEM allocation; the base address lands in *dst (shared).
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 TMEM lanes x 16 consecutive 32-bit columns: thread t of the warp receives
// lane (32*(warp%4) + t), columns [col, col+16).
__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ void ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}

// MMA with A from TMEM (lane = row m, 32-bit column = k) and B from shared memory.
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

// 32 TMEM lanes x 16 columns from registers (thread t of the warp -> lane 32*(warp%4) + t).
__device__ __forceinline__ void st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MN-major operand in the SWIZZLE_128B_BASE32B layout (the MN-major form the
// tensor core accepts for 32-bit types): atoms of 4 K-rows x 128 B along MN,
// 32-byte chunks XOR-swizzled by the K-row; MN atoms `lbo` bytes apart, 4-row K
// groups `sbo` bytes apart. Element (mn, k) of such a tile, in floats, with
// `mn_atoms` = MN extent / 32; the tile must be 512-byte aligned.
__device__ __forceinline__ int mn32_idx(int mn, int k, int mn_atoms) {
    return ((mn >> 5) << 7) + (k >> 2) * (mn_atoms << 7) + ((k & 3) << 5) + (((((mn & 31) >> 3) ^ (k & 3))) << 3) +
           (mn & 7);
}
__device__ __forceinline__ uint64_t mn32_desc(const float* tile, int mn_atoms) {
    return sdesc(tile, 512u, static_cast<uint32_t>(mn_atoms) * 512u) | (1ull << 61);  // layout 1: 128B_BASE32B
}

// K-major SWIZZLE_128B operand (the layout a TMA tensor load with
// CU_TENSOR_MAP_SWIZZLE_128B and a 32-float box width writes): per 32-element K
// block, rows of 128 B with their 16-byte chunks XOR-swizzled by row % 8, 8-row
// groups 1024 B apart. `p` is the K-step's start: block base + (k % 32) floats;
// the block base must be 1024-byte aligned.
__device__ __forceinline__ uint64_t sw128_desc(const float* p) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr(p) >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1) << 16;          // LBO: unused for swizzled K-major
    d |= static_cast<uint64_t>(1024 >> 4) << 32;  // SBO: 8 rows x 128 B
    d |= static_cast<uint64_t>(1) << 46;          // descriptor version (sm100)
    d |= static_cast<uint64_t>(2) << 61;          // SWIZZLE_128B
    return d;
}
// K-step s (8 elements) of a [rows][KW] SW128 tile stored as KW/32 blocks of rows x 32.
__device__ __forceinline__ uint64_t sw128_kdesc(const float* tile, int s, int rows) {
    return sw128_desc(tile + (s >> 2) * rows * 32 + (s & 3) * 8);
}

// TMA: 2D tile of a tensor map into shared memory, completion on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            saddr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(saddr(bar))
        : "memory");
}

// The tensor core reads a kind::tf32 operand's 32-bit container as tf32 by
// TRUNCATION (measured: scratch/sw128_test.cu), so raw fp32 data in shared
// memory is a valid "hi" operand and lo = x - trunc_tf32(x) completes the split.
__device__ __forceinline__ float tf32_trunc_lo(float x) {
    return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// fp32 -> (tf32 hi, fp32 lo) split for 3xTF32.
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    hi = __uint_as_float(h);
    lo = x - hi;
}

}  // namespace umma
}  // namespace lamm_b200
