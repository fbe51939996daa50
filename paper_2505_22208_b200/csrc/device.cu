// device.cu - host orchestration of the sm_100a LaMM step: lamm_ctx, device
// buffers, batch staging, the captured CUDA graph of the step, NCCL, and the
// device half of the C ABI declared in include/lamm_b200.h.
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.hpp"
#include "edge_kernels.cuh"
#include "kernels.cuh"
#include "gemm_kernels.cuh"
#include "rng.hpp"

namespace lamm_b200 {

#define CK(x)                                                                                        \
    do {                                                                                             \
        const cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) throw CudaErr(std::string(#x) + ": " + cudaGetErrorString(e_));       \
    } while (0)

// ---------------------------------------------------------------- NCCL ----
// Loaded at first use so the library has no link-time NCCL dependency and
// binds whichever libnccl.so.2 the process already has (torch's or the system's).
struct NcclApi {
    bool ok = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy && a.error_string;
        return a;
    }();
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw NcclErr(std::string(what) + ": " + nccl().error_string(r));
}

// ------------------------------------------------------------- buffers ----
struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct KernelSlot {
    std::string name;
    cudaEvent_t a = nullptr, b = nullptr;
};

struct Ops;

}  // namespace lamm_b200

struct lamm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    lamm_model_config cfg{};
    int H = 0, L = 0, K = 0, D = 0;
    int64_t NP = 0;
    int nsm = 148;
    const lamm_b200::Ops* ops = nullptr;
    // persistent parameter state
    lamm_b200::Buf p64, v64, g64, p32, tanh_emb, grads, block_scratch, wpack;
    // TMA descriptors of the [Ncap][H] activation buffers the node GEMMs read,
    // by base address (rebuilt when ensure_capacity reallocates)
    std::map<const void*, CUtensorMap> tmaps;
    // staging (pinned host -> device blob, header first)
    char* h_stage = nullptr;
    size_t h_stage_cap = 0;
    lamm_b200::Buf d_stage;
    lamm_b200::Buf d_stage_alt;  // the other batch-state parity's staging blob (neighbour-list pipelining)
    lamm_b200::StepHeader* h_result = nullptr;  // pinned copy of the header after a step
    // capacities
    int64_t Ncap = 0, Bcap = 0, Pcap = 0;
    std::map<std::string, lamm_b200::Buf> bufs;
    // reference table
    bool use_table = false;
    int ntab = 0;
    std::vector<uint8_t> h_thas;
    // host mirror of the current batch
    int32_t B = 0;
    int64_t N = 0;
    int n_large = 0;  // samples of the current batch counted by k_cell_count
    bool omit_cell_count = false;  // set while capturing g_full[0] (batches with n_large == 0)
    std::vector<int64_t> h_atom_ptr;
    std::vector<int32_t> h_Z, h_dsidx;
    std::vector<uint8_t> h_emask, h_fmask;
    int me = 0, mf = 0;
    bool batch_valid = false, nlist_valid = false, fwd_valid = false, loss_valid = false;
    bool grads_in_acc = false;  // the last step was lamm_train_step_workers: its worker sum is in g64
    // launch geometry
    int grid_warp = 0, grid_gemm = 0, grid_upd = 0, grid_small = 0, grid_opt = 0, ncta_red = 0, grid_reduce = 0;
    int grid_edge = 0, grid_emb = 0;
    // graphs
    cudaGraphExec_t g_step = nullptr, g_opt = nullptr;
    // step (+ allreduce) + optimizer in one graph; [1]: with k_cell_count (batches with
    // samples above kSmallAtoms or periodic ones), [0]: without
    cudaGraphExec_t g_full[2] = {nullptr, nullptr};
    // neighbour-list pipelining (lamm_train_step_staged_next): the batch state that
    // k_prep / k_cell_count / k_nbr_fill write exists twice; step k's model runs on one
    // parity while the next step's neighbour list is built into the other on `side`.
    // swap_parity() exchanges the two sets (buffers, staging blob, graphs).
    cudaGraphExec_t g_nl[2] = {nullptr, nullptr}, g_model = nullptr;
    struct ParityGraphs {
        cudaGraphExec_t g_full[2] = {nullptr, nullptr}, g_nl[2] = {nullptr, nullptr}, g_model = nullptr,
                        g_step = nullptr, g_opt = nullptr;
    } alt_graphs;
    bool pipe_alloc = false, pipe_valid = false;
    int pipe_slot = -1, par = 0;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_prev = nullptr, ev_nl = nullptr;
    bool graph_dirty = true;
    bool use_graph = true, profile = false, export64 = false, pdl = true;
    bool rank_local = false;  // option "rank_local": workers > 1 without a communicator (one rank's share only)
    int denoise_scheme = 1;
    double opt_inv_g = 1.0, opt_lr = 0, opt_decay = 0, opt_eps = 0, opt_clip = 0;
    int opt_G = 1;
    // device-resident staged batches (lamm_stage)
    struct Slot {
        lamm_b200::Buf blob;
        size_t bytes = 0;
        int32_t B = 0;
        int64_t N = 0;
        int me = 0, mf = 0, n_large = 0;
    };
    std::vector<Slot> staged;
    // pipelined steps (lamm_train_step_submit / _wait): at most two in flight,
    // each with its own pinned blob and pinned result header
    struct Inflight {
        char* blob = nullptr;
        size_t cap = 0, bytes = 0;
        lamm_b200::Buf inbox;          // device copy of the blob, uploaded on copy_stream
        cudaEvent_t uploaded = nullptr;
        lamm_b200::StepHeader* result = nullptr;
        cudaEvent_t done = nullptr;
        cudaEvent_t nl_done = nullptr;  // its batch preparation finished (side stream)
        int32_t B = 0, workers = 1, rank = 0;
        int64_t N = 0, step = 0;
        int me = 0, mf = 0, n_large = 0;
        lamm_train_config tc{};
    };
    Inflight ring[2];
    cudaStream_t copy_stream = nullptr;  // uploads of pipelined steps (overlap the running step)
    int64_t next_ticket = 0, oldest_ticket = 0;
    lamm_b200::Buf anomaly, flush;
    // NCCL
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    // timing
    cudaEvent_t ev[64] = {};
    std::vector<lamm_b200::KernelSlot> slots;
    size_t slot_cursor = 0;
    std::map<std::string, std::pair<double, int64_t>> ktimes;
    int64_t launches = 0, last_step_launches = 0, graph_launches = 0;
    int flush_flip = 0;
    // per-step device intervals (upload -> optimizer): a ring of event pairs, so steps
    // submitted without a sync are timed too; collected in order once complete
    static constexpr int kStepRing = 64;
    cudaEvent_t step_ev[kStepRing][2] = {};
    int ring_next = 0, last_slot = -1;
    std::vector<int> ring_pending;
    cudaEvent_t coll_ev = nullptr;  // recorded inside the step just before the gradient allreduce
    double compute_ms_last = -1.0;  // upload -> allreduce of the last synced step (communicator only)
    double step_ms_total = 0.0;
    int64_t step_count = 0;
    int64_t last_h2d = 0;
};

namespace lamm_b200 {

using Ctx = lamm_ctx;

// Entry points that touch the device state refuse to run while pipelined steps
// (lamm_train_step_submit) are in flight.
// A prefetched neighbour list (lamm_train_step_staged_next) may still be building
// into the other batch-state parity on the side stream: finish it and forget it.
void drain_pipe(Ctx& c) {
    if (c.side) CK(cudaStreamSynchronize(c.side));
    c.pipe_valid = false;
}
// keep_prefetch: the call touches only the parameter / optimizer / gradient state,
// which the batch preparation neither reads nor writes — a prefetched batch stays valid.
void require_no_chain(Ctx& c, bool keep_prefetch = false) {
    require(c.oldest_ticket == c.next_ticket, "call while pipelined steps are in flight (lamm_train_step_wait first)");
    if (!keep_prefetch) drain_pipe(c);
}

Buf& buf(Ctx& c, const std::string& name) { return c.bufs[name]; }

// The batch state: everything k_prep / k_cell_count / k_nbr_fill write and the model
// kernels read. With pipelining on, each has a second copy ("<name>#1").
bool is_batch_state(const std::string& n) {
    static const char* const names[] = {"atom_ptr", "Z",    "zslot",  "z2s",  "dsidx", "emask",   "fmask",  "denoise",
                                        "sample_of", "chan", "x",      "y",    "z",     "En",      "Fn",     "cnt",
                                        "lptr",     "stot", "soff",   "row_ptr", "col", "dst",     "colz",   "segw",
                                        "geo",      "rbf",  "rbfl",   "rbfp", "part_lo", "cgrid",  "acell",  "cstart",
                                        "cpos",     "sdone", "cmask", "fw",   "dist64", "unit64"};
    for (const char* k : names)
        if (n == k) return true;
    return false;
}

void ensure_one(Ctx& c, const std::string& name, size_t bytes, bool& changed) {
    Buf& b = c.bufs[name];
    if (b.bytes >= bytes && b.p) return;
    if (b.p) CK(cudaFree(b.p));
    b.p = nullptr;
    CK(cudaMalloc(&b.p, std::max<size_t>(bytes, 256)));
    b.bytes = std::max<size_t>(bytes, 256);
    changed = true;
}

void ensure_buf(Ctx& c, const std::string& name, size_t bytes, bool& changed) {
    ensure_one(c, name, bytes, changed);
    if (c.pipe_alloc && is_batch_state(name)) ensure_one(c, name + "#1", bytes, changed);
}

// Exchanges the two batch-state parities: buffers, staging blob and the graphs
// captured over them (the rest of the code always works on "the current" set).
void swap_parity(Ctx& c) {
    for (auto& kv : c.bufs) {
        const std::string& n = kv.first;
        if (n.size() > 2 && n.compare(n.size() - 2, 2, "#1") == 0) continue;
        if (!is_batch_state(n)) continue;
        auto it = c.bufs.find(n + "#1");
        if (it != c.bufs.end()) std::swap(kv.second, it->second);
    }
    std::swap(c.d_stage, c.d_stage_alt);
    auto& a = c.alt_graphs;
    std::swap(c.g_full[0], a.g_full[0]);
    std::swap(c.g_full[1], a.g_full[1]);
    std::swap(c.g_nl[0], a.g_nl[0]);
    std::swap(c.g_nl[1], a.g_nl[1]);
    std::swap(c.g_model, a.g_model);
    std::swap(c.g_step, a.g_step);
    std::swap(c.g_opt, a.g_opt);
    c.par ^= 1;
}

void alloc_param_state(Ctx& c) {
    auto mk = [&](Buf& b, size_t bytes) {
        CK(cudaMalloc(&b.p, bytes));
        CK(cudaMemset(b.p, 0, bytes));
        b.bytes = bytes;
    };
    mk(c.p64, sizeof(double) * c.NP);
    mk(c.v64, sizeof(double) * c.NP);
    mk(c.g64, sizeof(double) * (c.NP + 4));
    mk(c.p32, sizeof(float) * c.NP);
    mk(c.tanh_emb, sizeof(float) * kMaxZ * c.H);
    mk(c.grads, sizeof(float) * (c.NP + 4));
    mk(c.block_scratch, sizeof(double) * 4096);
    mk(c.anomaly, 256);
    mk(c.wpack, sizeof(float) * 4 * c.H * c.H * std::max(c.L, 1));
}

// Grows every batch-sized buffer to hold N atoms, B samples and P pairs.
void ensure_capacity(Ctx& c, int64_t N, int64_t B, int64_t P) {
    bool changed = false;
    if (N > c.Ncap) c.Ncap = std::max<int64_t>(N + N / 4, 1024);
    if (B > c.Bcap) c.Bcap = std::max<int64_t>(B + B / 4, 64);
    if (P > c.Pcap) c.Pcap = std::max<int64_t>(P + P / 4, 4096);
    const int64_t Nc = c.Ncap, Bc = c.Bcap, Pc = c.Pcap;
    const int H = c.H, K = c.K, D = c.D, L = c.L;
    ensure_buf(c, "atom_ptr", 8 * (Bc + 1), changed);
    ensure_buf(c, "Z", 4 * Nc, changed);
    ensure_buf(c, "zslot", 4 * Nc, changed);
    ensure_buf(c, "z2s", 4 * 128, changed);
    ensure_buf(c, "dsidx", 4 * Bc, changed);
    ensure_buf(c, "emask", Bc, changed);
    ensure_buf(c, "fmask", Bc, changed);
    ensure_buf(c, "denoise", Bc, changed);
    ensure_buf(c, "sample_of", 4 * Nc, changed);
    ensure_buf(c, "chan", 4 * Nc, changed);
    for (const char* n : {"x", "y", "z"}) ensure_buf(c, n, 8 * Nc, changed);
    ensure_buf(c, "En", 8 * Bc, changed);
    ensure_buf(c, "Fn", 24 * Nc, changed);
    ensure_buf(c, "cnt", 4 * Nc, changed);
    ensure_buf(c, "lptr", 4 * Nc, changed);
    ensure_buf(c, "stot", 4 * Bc, changed);
    ensure_buf(c, "soff", 4 * Bc, changed);
    ensure_buf(c, "row_ptr", 4 * (Nc + 1), changed);
    const int64_t Pp = ((Pc + kChunk + 16 + 7) / 8) * 8;  // CSR padding for the chunk staging
    ensure_buf(c, "col", 4 * Pp, changed);
    ensure_buf(c, "dst", 4 * Pp, changed);
    ensure_buf(c, "colz", 4 * Pp, changed);
    ensure_buf(c, "segw", 4 * (Pp / 32 + 32), changed);
    ensure_buf(c, "geo", 16 * Pp, changed);
    ensure_buf(c, "sij", 8 * Pp, changed);
    ensure_buf(c, "rbf", 4 * static_cast<size_t>(Pp) * K, changed);
    ensure_buf(c, "rbfl", 4 * static_cast<size_t>(Pp) * K, changed);
    ensure_buf(c, "rbfp", 4 * static_cast<size_t>(Pp) * K, changed);
    ensure_buf(c, "part_lo", 4 * (static_cast<size_t>(c.grid_edge) * kPartsPerCta + 1), changed);
    ensure_buf(c, "cgrid", sizeof(CellGrid) * Bc, changed);
    ensure_buf(c, "acell", 4 * Nc, changed);
    ensure_buf(c, "cstart", 4 * (4 * Nc + 65 * Bc + 1), changed);
    ensure_buf(c, "cpos", 32 * Nc, changed);
    ensure_buf(c, "sdone", 4 * Bc, changed);
    ensure_buf(c, "cmask", 4 * kMaskWords * Nc, changed);
    ensure_buf(c, "eatom", 8 * Nc, changed);
    ensure_buf(c, "fterm", 8 * Nc, changed);
    ensure_buf(c, "fw", 8 * Nc, changed);
    if (c.export64) {
        ensure_buf(c, "dist64", 8 * Pc, changed);
        ensure_buf(c, "unit64", 24 * Pc, changed);
    }
    for (int l = 1; l <= L; ++l) {
        ensure_buf(c, "t" + std::to_string(l), 4 * static_cast<size_t>(Nc) * H, changed);
        ensure_buf(c, "h" + std::to_string(l), 4 * static_cast<size_t>(Nc) * H, changed);
    }
    for (int l = 0; l < L; ++l) ensure_buf(c, "mu" + std::to_string(l), 4 * static_cast<size_t>(Nc) * H, changed);
    ensure_buf(c, "F", 12 * Nc * D, changed);
    ensure_buf(c, "Yf", 4 * static_cast<size_t>(Nc) * ((3 * H + 3 + 3 * K + 3) / 4 * 4), changed);  // ForceBody::kYW
    ensure_buf(c, "Epred", 8 * Bc * D, changed);
    ensure_buf(c, "gE", 4 * Bc * D, changed);
    ensure_buf(c, "gF", 12 * Nc * D, changed);
    ensure_buf(c, "gFc", 16 * Nc, changed);
    ensure_buf(c, "sample_terms", 16 * Bc, changed);
    ensure_buf(c, "gh", 4 * static_cast<size_t>(Nc) * H, changed);
    ensure_buf(c, "gm", 4 * static_cast<size_t>(Nc) * H, changed);
    for (int l = 0; l < L; ++l) {
        ensure_buf(c, "part_wf" + std::to_string(l), 4 * static_cast<size_t>(c.grid_edge) * H * K, changed);
        ensure_buf(c, "part_wu" + std::to_string(l),
                   4 * static_cast<size_t>(std::max(c.grid_gemm, c.grid_upd)) * H * H, changed);
    }
    ensure_buf(c, "part_head", 4 * static_cast<size_t>(c.grid_edge) * (3 * H + K) * D, changed);
    ensure_buf(c, "part_emb", 4 * static_cast<size_t>(c.grid_emb) * kMaxZ * H, changed);
    if (changed) {
        c.graph_dirty = true;
        c.tmaps.clear();
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// TMA map of an fp32 [Ncap][H] activation buffer: 32 x 128 boxes (one 128-atom
// tile's K block), SWIZZLE_128B, the layout umma::sw128_desc describes.
CUtensorMap act_map(Ctx& c, const float* base) {
    auto it = c.tmaps.find(base);
    if (it != c.tmaps.end()) return it->second;
    CUtensorMap m{};
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(c.H), static_cast<cuuint64_t>(c.Ncap)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(c.H) * 4};
    const cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    c.tmaps[base] = m;
    return m;
}

Dev make_dev(Ctx& c) {
    Dev d{};
    d.H = c.H, d.L = c.L, d.K = c.K, d.D = c.D;
    d.rc = c.cfg.cutoff;
    d.Ncap = c.Ncap, d.Bcap = c.Bcap, d.Pcap = c.Pcap;
    d.hdr = c.d_stage.as<StepHeader>();
    d.atom_ptr = buf(c, "atom_ptr").as<int64_t>();
    d.Z = buf(c, "Z").as<int32_t>();
    d.zslot = buf(c, "zslot").as<int32_t>();
    d.z_to_slot = buf(c, "z2s").as<int32_t>();
    d.dsidx = buf(c, "dsidx").as<int32_t>();
    d.emask = buf(c, "emask").as<uint8_t>();
    d.fmask = buf(c, "fmask").as<uint8_t>();
    d.denoise = buf(c, "denoise").as<uint8_t>();
    d.sample_of = buf(c, "sample_of").as<int32_t>();
    d.chan = buf(c, "chan").as<int32_t>();
    d.x = buf(c, "x").as<double>(), d.y = buf(c, "y").as<double>(), d.z = buf(c, "z").as<double>();
    d.En = buf(c, "En").as<double>();
    d.Fn = buf(c, "Fn").as<double>();
    d.use_table = c.use_table ? 1 : 0;
    d.denoise_scheme = c.denoise_scheme;
    d.ntab = c.ntab;
    d.rho = buf(c, "rho").as<double>();
    d.rho_has = buf(c, "rho_has").as<uint8_t>();
    d.tmean = buf(c, "tmean").as<double>();
    d.tstd = buf(c, "tstd").as<double>();
    d.tfstd = buf(c, "tfstd").as<double>();
    d.thas = buf(c, "thas").as<uint8_t>();
    d.cnt = buf(c, "cnt").as<int32_t>();
    d.lptr = buf(c, "lptr").as<int32_t>();
    d.stot = buf(c, "stot").as<int32_t>();
    d.soff = buf(c, "soff").as<int32_t>();
    d.row_ptr = buf(c, "row_ptr").as<int32_t>();
    d.segw = buf(c, "segw").as<uint32_t>();
    d.col = buf(c, "col").as<int32_t>();
    d.dst = buf(c, "dst").as<int32_t>();
    d.colz = buf(c, "colz").as<int32_t>();
    d.part_lo = buf(c, "part_lo").as<int32_t>();
    d.cgrid = buf(c, "cgrid").as<CellGrid>();
    d.acell = buf(c, "acell").as<int32_t>();
    d.cstart = buf(c, "cstart").as<int32_t>();
    d.cpos = buf(c, "cpos").as<double4>();
    d.sdone = buf(c, "sdone").as<uint32_t>();
    d.cmask = buf(c, "cmask").as<uint32_t>();
    d.eatom = buf(c, "eatom").as<double>();
    d.fterm = buf(c, "fterm").as<double>();
    d.fw = buf(c, "fw").as<double>();
    d.geo = buf(c, "geo").as<float4>();
    d.sij = buf(c, "sij").as<float2>();
    d.rbf = buf(c, "rbf").as<float>();
    d.rbfl = buf(c, "rbfl").as<float>();
    d.rbfp = buf(c, "rbfp").as<float>();
    d.export64 = c.export64 ? 1 : 0;
    d.dist64 = c.export64 ? buf(c, "dist64").as<double>() : nullptr;
    d.unit64 = c.export64 ? buf(c, "unit64").as<double>() : nullptr;
    float* p = c.p32.as<float>();
    const int H = c.H, K = c.K, D = c.D, L = c.L;
    d.emb = p;
    p += kMaxZ * H;
    for (int l = 0; l < L; ++l) d.wf[l] = p, p += H * K;
    for (int l = 0; l < L; ++l) d.wu[l] = p, p += H * H;
    d.we = p, p += H * D;
    d.wfh = p;
    d.tanh_emb = c.tanh_emb.as<float>();
    d.tanh_emb_w = c.tanh_emb.as<float>();
    for (int l = 1; l <= L; ++l) {
        d.t[l] = buf(c, "t" + std::to_string(l)).as<float>();
        d.h[l] = buf(c, "h" + std::to_string(l)).as<float>();
    }
    for (int l = 0; l < L; ++l) d.mu[l] = buf(c, "mu" + std::to_string(l)).as<float>();
    d.F = buf(c, "F").as<float>();
    d.Yf = buf(c, "Yf").as<float>();
    d.Epred = buf(c, "Epred").as<double>();
    d.gE = buf(c, "gE").as<float>();
    d.gF = buf(c, "gF").as<float>();
    d.gFc = buf(c, "gFc").as<float4>();
    d.sample_terms = buf(c, "sample_terms").as<double>();
    d.block_scratch = c.block_scratch.as<double>();
    d.gh = buf(c, "gh").as<float>();
    d.gm = buf(c, "gm").as<float>();
    for (int l = 0; l < L; ++l) {
        d.part_wf[l] = buf(c, "part_wf" + std::to_string(l)).as<float>();
        d.part_wu[l] = buf(c, "part_wu" + std::to_string(l)).as<float>();
    }
    d.part_head = buf(c, "part_head").as<float>();
    d.part_emb = buf(c, "part_emb").as<float>();
    d.ncta_edge = c.grid_edge, d.ncta_gemm = c.grid_gemm, d.ncta_red = c.ncta_red;
    d.grads = c.grads.as<float>();
    d.p64 = c.p64.as<double>();
    d.v64 = c.v64.as<double>();
    d.g64_in = nullptr;
    d.g64_loss = 0;
    d.g64_acc = c.g64.as<double>();
    d.p32 = c.p32.as<float>();
    d.NP = c.NP;
    d.emb_rows = kMaxZ;
    d.anomaly = c.anomaly.as<unsigned int>();
    d.wpack = c.wpack.as<float>();
    return d;
}

BatchArrays make_batch_arrays(Ctx& c) {
    BatchArrays b{};
    b.atom_ptr = buf(c, "atom_ptr").as<int64_t>();
    b.Z = buf(c, "Z").as<int32_t>();
    b.zslot = buf(c, "zslot").as<int32_t>();
    b.z_to_slot = buf(c, "z2s").as<int32_t>();
    b.dsidx = buf(c, "dsidx").as<int32_t>();
    b.emask = buf(c, "emask").as<uint8_t>();
    b.fmask = buf(c, "fmask").as<uint8_t>();
    b.denoise = buf(c, "denoise").as<uint8_t>();
    return b;
}

// ------------------------------------------------------------- launches ---
// Timing experiments only, compiled in with -DLAMM_TIMING_KNOBS (never in the
// shipped build): LAMM_SKIP_KERNEL=<name> leaves that kernel out of the step
// (results are then wrong; used to measure a kernel's marginal cost).
#ifdef LAMM_TIMING_KNOBS
inline bool skipped(const char* name) {
    const char* s = std::getenv("LAMM_SKIP_KERNEL");
    return s != nullptr && std::strcmp(s, name) == 0;
}
#else
constexpr bool skipped(const char*) { return false; }
#endif

template <class Kern, class... Args>
void launch(Ctx& c, const char* name, Kern kernel, int grid, int block, size_t smem, Args... args) {
    if (skipped(name)) return;
    KernelSlot* slot = nullptr;
    if (c.profile) {
        if (c.slot_cursor >= c.slots.size()) {
            KernelSlot s;
            CK(cudaEventCreate(&s.a));
            CK(cudaEventCreate(&s.b));
            c.slots.push_back(s);
        }
        slot = &c.slots[c.slot_cursor++];
        slot->name = name;
        // External records become real event-record nodes under graph capture
        // (a plain record would only add a dependency edge).
        CK(cudaEventRecordWithFlags(slot->a, c.stream, cudaEventRecordExternal));
    }
    // programmatic dependent launch: the kernel calls pdl_enter() before it
    // touches the previous kernel's outputs (device.cuh)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = c.pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kernel, args...));
    if (slot) CK(cudaEventRecordWithFlags(slot->b, c.stream, cudaEventRecordExternal));
    ++c.launches;
}

// Cooperative launch (all CTAs co-resident, for kernels with grid barriers);
// capturable into the step graph like a plain launch.
template <class... KArgs, class... Args>
void launch_coop(Ctx& c, const char* name, void (*kernel)(KArgs...), int grid, int block, Args... args) {
    if (skipped(name)) return;
    KernelSlot* slot = nullptr;
    if (c.profile) {
        if (c.slot_cursor >= c.slots.size()) {
            KernelSlot s;
            CK(cudaEventCreate(&s.a));
            CK(cudaEventCreate(&s.b));
            c.slots.push_back(s);
        }
        slot = &c.slots[c.slot_cursor++];
        slot->name = name;
        CK(cudaEventRecordWithFlags(slot->a, c.stream, cudaEventRecordExternal));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr2[2];
    attr2[0].id = cudaLaunchAttributeCooperative;
    attr2[0].val.cooperative = 1;
    attr2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr2[1].val.programmaticStreamSerializationAllowed = c.pdl ? 1 : 0;
    cfg.attrs = attr2;
    cfg.numAttrs = 2;
    CK(cudaLaunchKernelEx(&cfg, kernel, args...));
    if (slot) CK(cudaEventRecordWithFlags(slot->b, c.stream, cudaEventRecordExternal));
    ++c.launches;
}

void collect_kernel_times(Ctx& c) {
    if (!c.profile) return;
    for (size_t k = 0; k < c.slot_cursor && k < c.slots.size(); ++k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c.slots[k].a, c.slots[k].b) == cudaSuccess) {
            auto& e = c.ktimes[c.slots[k].name];
            e.first += ms;
            e.second += 1;
        } else {
            (void)cudaGetLastError();
        }
    }
}

struct Ops {
    void (*setup)(Ctx&);
    void (*prep)(Ctx&);
    void (*nlist)(Ctx&);
    void (*forward)(Ctx&, bool energy);
    void (*loss)(Ctx&, bool energy);
    void (*backward)(Ctx&, bool general);
    void (*opt)(Ctx&, const Dev&, int G, double inv_g, double clip, double lr, double decay, double eps);
    void (*pack)(Ctx&);
};

template <int H, int K>
struct Model {
    using ES = EdgeKernelSmem<H, K>;
    static constexpr size_t kGemmSmem = NodeGemmSmem<H>::bytes;
    static constexpr size_t kDwuSmem = DwuSmem<H>::bytes;
    static constexpr bool kFusedBwd = H == 128;  // k_bwd_gemm: update backward + dW_u in one kernel
    static constexpr bool kFusedUpd = H == 128;  // k_message_update: message walk + the CTA's own update GEMM
    static size_t smem_message() { return ES::message(); }
    static size_t smem_force(int D) { return ES::force(D); }
    static size_t smem_head(int D) { return ES::head(D); }
    static size_t smem_bwd() { return ES::bwd(); }

    static void set_smem(const void* fn, size_t bytes) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    }

    static void setup(Ctx& c) {
        set_smem((const void*)k_node_gemm<H>, kGemmSmem);
        set_smem((const void*)k_dwu<H>, kDwuSmem);
        if constexpr (kFusedBwd) set_smem((const void*)k_bwd_gemm<H>, BwdGemmSmem<H>::bytes);
        set_smem((const void*)k_edge_message<H, K, true>, smem_message());
        set_smem((const void*)k_edge_message<H, K, false>, smem_message());
        if constexpr (kFusedUpd) {
            set_smem((const void*)k_message_update<K, true>, MsgUpdSmem<K>::bytes);
            set_smem((const void*)k_message_update<K, false>, MsgUpdSmem<K>::bytes);
        }
        int smem_max = 0;
        CK(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
        if (smem_head(c.D) > static_cast<size_t>(smem_max) || 3 * c.D > H)
            throw InputErr("model: too many heads for the device path at this hidden size");
        // embedding-gradient slots (distinct Z per device-batch) that fit next to the staging
        set_smem((const void*)k_edge_force<H, K>, smem_force(c.D));
        set_smem((const void*)k_edge_head<H, K, false>, smem_head(c.D));
        set_smem((const void*)k_edge_head<H, K, true>, smem_head(c.D));
        set_smem((const void*)k_edge_bwd<H, K, true>, smem_bwd());
        set_smem((const void*)k_edge_bwd<H, K, false>, smem_bwd());
        set_smem((const void*)k_emb_grad, sizeof(float) * kMaxZ * H);
        c.grid_emb = 4 * c.nsm;  // ~13 atoms per CTA at cfg2: the gh loads of a CTA in flight together
        // one tcgen05 CTA per SM, persistent over 128-atom tiles; a multiple of the
        // column split so a CTA keeps one column block (k_bwd_gemm's dW_u partials)
        c.grid_upd = c.nsm / NodeGemmCfg<H>::NS * NodeGemmCfg<H>::NS;
        c.grid_gemm = c.nsm / 2;       // split-K CTAs of dW_u (one partial each)
        // one edge partitioning (k_nbr_fill) serves all four edge kernels: size it so
        // every CTA of the heaviest one is resident (no second wave)
        int occ_e = 8, o = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_edge_message<H, K, false>, kMsgGroups * H, smem_message()));
        occ_e = std::min(occ_e, o);
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_edge_force<H, K>, kForceGroups * H, smem_force(c.D)));
        occ_e = std::min(occ_e, o);
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_edge_head<H, K, false>, kGroups * H, smem_head(c.D)));
        occ_e = std::min(occ_e, o);
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_edge_bwd<H, K, false>, kGroups * H, smem_bwd()));
        occ_e = std::min(occ_e, o);
        c.grid_edge = c.nsm * std::max(1, occ_e);
        c.grid_warp = 4 * c.nsm;
        c.grid_small = c.nsm * 4;
        c.ncta_red = c.nsm;
        c.grid_opt = static_cast<int>(std::min<int64_t>((c.NP + 255) / 256, std::min(c.nsm, 256)));  // cooperative, <= 256 CTAs
        c.grid_reduce = static_cast<int>(std::min<int64_t>((c.NP + 31) / 32, 16 * c.nsm));
    }

    static void prep(Ctx& c) {
        launch(c, "prep", k_prep, c.grid_small, 128, 0, make_dev(c), make_batch_arrays(c), c.grid_edge * kPartsPerCta);
    }

    static void nlist(Ctx& c) {
        const Dev d = make_dev(c);
        if (!c.omit_cell_count)  // (k_prep finalizes the CSR itself when no sample needs k_cell_count)
            launch(c, "cell_count", k_cell_count, 2 * c.nsm, 256, 0, d, c.grid_edge * kPartsPerCta);  // one wave
        launch(c, "nbr_fill", k_nbr_fill<K>, c.grid_warp, 256, 0, d, c.grid_edge * kPartsPerCta);
    }

    // energy = false leaves the per-sample energies to the fused loss kernel.
    static void forward(Ctx& c, bool energy) {
        const Dev d = make_dev(c);
        if (c.L == 0) throw InputErr("model: layers == 0 is not supported by the device path");
        for (int l = 0; l < c.L; ++l) {
            if constexpr (kFusedUpd) {  // one kernel per layer: message walk + the CTA's own update GEMM
                launch(c, "message", l == 0 ? k_message_update<K, true> : k_message_update<K, false>, c.grid_edge,
                       kMsgGroups * H, MsgUpdSmem<K>::bytes, d, l);
                continue;
            }
            launch(c, "message", l == 0 ? k_edge_message<H, K, true> : k_edge_message<H, K, false>, c.grid_edge,
                   kMsgGroups * H, smem_message(), d, l);
            launch(c, "update", k_node_gemm<H>, c.grid_upd, NodeGemmCfg<H>::NT, kGemmSmem, d, l, 0, act_map(c, d.mu[l]),
                   act_map(c, d.h[l + 1]), act_map(c, d.t[l + 1]));
        }
        launch(c, "force", k_edge_force<H, K>, c.grid_edge, kForceGroups * H, smem_force(c.D), d);
        launch(c, "force_out", k_force_out<H, K>, 2 * c.nsm, 256, 0, d, energy ? 0 : 1);  // fewer CTAs: each stages the head weights
        if (energy) launch(c, "energy", k_energy, c.grid_small, 128, sizeof(double) * 128 * c.D, d);
    }

    static void loss(Ctx& c, bool energy) {
        const Dev d = make_dev(c);
        // the train step (energy fused here) only needs the compact per-atom force gradient
        // (with k_force_out's per-atom energies and force terms: forward(c, false))
        launch(c, "loss", k_loss, c.grid_small, 128, 0, d, energy ? 2 : 0, energy ? 0 : 1);
    }

    static void backward(Ctx& c, bool general) {
        const Dev d = make_dev(c);
        const int passes = general ? c.D : 1;
        for (int q = 0; q < passes; ++q)
            launch(c, "head_bwd", general ? k_edge_head<H, K, false> : k_edge_head<H, K, true>, c.grid_edge,
                   kGroups * H, smem_head(c.D), d, general ? q : -1,
                   q == 0 ? 1 : 0);
        for (int l = c.L - 1; l >= 0; --l) {
            if constexpr (kFusedBwd) {
                launch(c, "bwd_gemm", k_bwd_gemm<H>, c.grid_upd, 512, BwdGemmSmem<H>::bytes, d, l, act_map(c, d.gh));
            } else {
                launch(c, "bwd_gemm", k_node_gemm<H>, c.grid_upd, NodeGemmCfg<H>::NT, kGemmSmem, d, l, 1, act_map(c, d.gh),
                       act_map(c, d.gm), act_map(c, d.gm));
                launch(c, "dwu", k_dwu<H>, c.grid_gemm, 256, kDwuSmem, d, l);
            }
            launch(c, "bwd_edge", l == 0 ? k_edge_bwd<H, K, true> : k_edge_bwd<H, K, false>, c.grid_edge,
                   kGroups * H, smem_bwd(), d, l);
        }
        SegTable tab{};
        int64_t off = 0;
        auto add = [&](int64_t n, int kind, const float* src, int ncta, int stride) {
            tab.s[tab.nseg++] = Seg{off, static_cast<int32_t>(n), kind, src, ncta, stride};
            off += n;
        };
        launch(c, "emb_grad", k_emb_grad, c.grid_emb, 128, sizeof(float) * kMaxZ * H, d);
        add(static_cast<int64_t>(kMaxZ) * H, 1, d.part_emb, c.grid_emb, 0);
        for (int l = 0; l < c.L; ++l) add(H * K, 0, d.part_wf[l], c.grid_edge, H * K);
        for (int l = 0; l < c.L; ++l) {
            if constexpr (kFusedBwd)  // CTA c holds column block c % NS as [H][NC]
                add(H * H, 2, d.part_wu[l], c.grid_upd, H * NodeGemmCfg<H>::NC);
            else
                add(H * H, 0, d.part_wu[l], c.grid_gemm, H * H);
        }
        const int hw = (3 * H + K) * c.D;
        add(H * c.D, 0, d.part_head + (2 * H + K) * c.D, c.grid_edge, hw);
        add((2 * H + K) * c.D, 0, d.part_head, c.grid_edge, hw);
        launch(c, "grad_reduce", k_grad_reduce, c.grid_reduce, 256, 0, d, tab);
    }

    static void opt(Ctx& c, const Dev& d, int G, double inv_g, double clip, double lr, double decay, double eps) {
        launch_coop(c, "optimizer", k_opt<H>, c.grid_opt, 256, d, G, inv_g, clip, lr, decay, eps);
    }

    // Packs the tensor-core weight operands from the fp32 working parameters.
    static void pack(Ctx& c) {
        launch(c, "pack_weights", k_pack_weights<H>, 2 * c.nsm, 256, 0, make_dev(c));
    }

    static constexpr Ops ops{setup, prep, nlist, forward, loss, backward, opt, pack};
};

const Ops* select_ops(int H, int K) {
    if (H == 128 && K == 16) return &Model<128, 16>::ops;
    if (H == 128 && K == 8) return &Model<128, 8>::ops;
    if (H == 64 && K == 16) return &Model<64, 16>::ops;
    if (H == 64 && K == 8) return &Model<64, 8>::ops;
    if (H == 32 && K == 8) return &Model<32, 8>::ops;
    if (H == 32 && K == 16) return &Model<32, 16>::ops;
    return nullptr;
}

// ------------------------------------------------------------- staging ----
inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

void ensure_stage(Ctx& c, size_t bytes) {
    if (bytes > c.h_stage_cap) {
        if (c.h_stage) CK(cudaFreeHost(c.h_stage));
        const size_t cap = bytes + bytes / 4 + 4096;
        CK(cudaMallocHost(reinterpret_cast<void**>(&c.h_stage), cap));
        c.h_stage_cap = cap;
    }
    for (Buf* st : {&c.d_stage, &c.d_stage_alt}) {
        if (st == &c.d_stage_alt && !c.pipe_alloc) continue;
        if (bytes <= st->bytes) continue;
        if (st->p) CK(cudaFree(st->p));
        const size_t cap = bytes + bytes / 4 + 4096;
        CK(cudaMalloc(&st->p, cap));
        st->bytes = cap;
        c.graph_dirty = true;
    }
}

// Validates a device-batch like the reference does (validate_system,
// validate_labels, masked_loss shape checks) and records the host mirror.
void validate_batch(Ctx& c, const lamm_batch_view* b) {
    require(b != nullptr && b->atom_ptr && b->positions && b->atomic_numbers, "batch: null arrays");
    require(b->n_samples >= 1, "batch: no samples");
    require(b->atom_ptr[0] == 0 && b->atom_ptr[b->n_samples] == b->n_atoms, "batch: atom_ptr/n_atoms mismatch");
    require(b->n_atoms < (int64_t(1) << 31), "batch: too many atoms for one device-batch");
    for (int32_t s = 0; s < b->n_samples; ++s) {
        require(b->atom_ptr[s + 1] > b->atom_ptr[s], "system has no atoms");
        const int d = b->dataset_index ? b->dataset_index[s] : 0;
        require(d >= 0, "negative dataset index");
        require(d < c.D, "masked_loss: dataset index outside prediction heads");
        if (c.use_table) require(d < c.ntab, "dataset index outside reference table");
    }
    for (int64_t k = 0; k < 3 * b->n_atoms; ++k) require(std::isfinite(b->positions[k]), "non-finite coordinate");
    for (int64_t a = 0; a < b->n_atoms; ++a)
        require(b->atomic_numbers[a] >= 1 && b->atomic_numbers[a] <= kMaxZ, "atomic number outside [1, 118]");
}

// Packs [StepHeader | atom_ptr | pos | Z | z2s | dsidx | emask | fmask | denoise
// | E | F | noise] into the pinned blob; returns its size. Effective masks:
// denoising samples train forces only (make_denoising_sample).
size_t pack_batch(Ctx& c, const lamm_batch_view* b, bool apply_denoise, const lamm_train_config* tc, int64_t step,
                  int32_t rank) {
    const int32_t B = b->n_samples;
    const int64_t N = b->n_atoms;
    bool any_dn = false;
    if (apply_denoise && b->denoise)
        for (int32_t s = 0; s < B; ++s) any_dn |= b->denoise[s] != 0;
    StepHeader h{};
    size_t off = align16(sizeof(StepHeader));
    auto place = [&](int64_t& field, size_t bytes) {
        field = static_cast<int64_t>(off);
        off = align16(off + bytes);
    };
    place(h.off_atom_ptr, 8 * (B + 1));
    place(h.off_pos, 24 * N);
    place(h.off_Z, 4 * N);
    place(h.off_z2s, 4 * 119);
    place(h.off_dsidx, 4 * B);
    place(h.off_emask, B);
    place(h.off_fmask, B);
    place(h.off_denoise, B);
    place(h.off_E, 8 * B);
    place(h.off_F, 24 * N);
    if (any_dn) place(h.off_noise, 24 * N);
    else h.off_noise = h.off_F;
    if (b->cell) place(h.off_cell, 8 * kCellDoubles * B);
    else h.off_cell = 0;
    h.blob_bytes = static_cast<int64_t>(off);
    ensure_stage(c, off);
    char* base = c.h_stage;
    std::memcpy(base + h.off_atom_ptr, b->atom_ptr, 8 * (B + 1));
    std::memcpy(base + h.off_pos, b->positions, 24 * N);
    std::memcpy(base + h.off_Z, b->atomic_numbers, 4 * N);
    int32_t* z2s = reinterpret_cast<int32_t*>(base + h.off_z2s);
    std::fill(z2s, z2s + 119, -1);
    int nslots = 0;
    for (int64_t a = 0; a < N; ++a)
        if (z2s[b->atomic_numbers[a]] < 0) z2s[b->atomic_numbers[a]] = nslots++;
    int32_t* ds = reinterpret_cast<int32_t*>(base + h.off_dsidx);
    uint8_t* em = reinterpret_cast<uint8_t*>(base + h.off_emask);
    uint8_t* fm = reinterpret_cast<uint8_t*>(base + h.off_fmask);
    uint8_t* dn = reinterpret_cast<uint8_t*>(base + h.off_denoise);
    double* E = reinterpret_cast<double*>(base + h.off_E);
    double* F = reinterpret_cast<double*>(base + h.off_F);
    int me = 0, mf = 0;
    for (int32_t s = 0; s < B; ++s) {
        ds[s] = b->dataset_index ? b->dataset_index[s] : 0;
        const bool is_dn = any_dn && b->denoise[s];
        dn[s] = is_dn ? 1 : 0;
        em[s] = is_dn ? 0 : (b->energy_mask ? b->energy_mask[s] : 0);
        fm[s] = is_dn ? 1 : (b->force_mask ? b->force_mask[s] : 0);
        require(!em[s] || b->energy, "energy mask set but energy missing");
        require(!(fm[s] && !is_dn) || b->forces, "force mask set but force rows != atom count");
        if (em[s] && c.use_table)
            require(c.h_thas[ds[s]] != 0, "normalize_labels: dataset has no fitted energy statistics");
        E[s] = em[s] ? b->energy[s] : 0.0;
        me += em[s], mf += fm[s];
    }
    if (b->forces) std::memcpy(F, b->forces, 24 * N);
    else std::memset(F, 0, 24 * N);
    if (b->cell) {  // {flag, cell, cell^-1, m[3], nimg} per sample (device.cuh: kCellDoubles)
        double* cs = reinterpret_cast<double*>(base + h.off_cell);
        for (int32_t s = 0; s < B; ++s) {
            const double* m = b->cell + 9 * static_cast<int64_t>(s);
            double* o = cs + static_cast<int64_t>(kCellDoubles) * s;
            bool periodic = false;
            for (int k = 0; k < 9; ++k) periodic |= m[k] != 0.0;
            std::memset(o, 0, sizeof(double) * kCellDoubles);
            if (!periodic) continue;
            for (int k = 0; k < 9; ++k) require(std::isfinite(m[k]), "cell: non-finite entry");
            require(cell_inverse(m, o + 10), "cell: singular");
            // images per axis: m_k = floor(1/2 + rc b_k (1 + 1e-9)), b_k = |column k of
            // cell^-1| = 1 / perpendicular width k (oracle/lamm_oracle.c:lor_image_range);
            // -1 on an open axis (pbc[k] = 0)
            const double* ci = o + 10;
            int nimg = 1;
            bool multi = false;
            for (int k = 0; k < 3; ++k) {
                const uint8_t* pb = b->pbc ? b->pbc + 3 * static_cast<int64_t>(s) : nullptr;
                int mk = -1;
                if (!pb || pb[k]) {
                    const double bk = std::sqrt((ci[k] * ci[k] + ci[3 + k] * ci[3 + k]) + ci[6 + k] * ci[6 + k]);
                    const double mm = std::floor(0.5 + c.cfg.cutoff * bk * (1.0 + 1e-9));
                    require(mm <= kMaxImages, "cell: far narrower than the cutoff (too many images)");
                    mk = static_cast<int>(mm);
                }
                o[19 + k] = static_cast<double>(mk);
                multi |= mk != 0;
                nimg *= 2 * std::max(mk, 0) + 1;
                require(nimg <= kMaxImages, "cell: more than 4096 images per pair (cell far narrower than the cutoff)");
            }
            o[22] = static_cast<double>(nimg);
            o[0] = multi ? 2.0 : 1.0;
            std::memcpy(o + 1, m, sizeof(double) * 9);
        }
    }
    if (any_dn) {
        // Raw displacement draws of make_denoising_sample: Rng(seed').normal(0, sigma)
        // per atom, x, y, z in order (S/denoise.cpp:31-40), with
        // seed' = mix_seed(mix_seed(seed, kNoiseTag + step), rank*B + b) (S/trainer.cpp:276-277).
        require(tc->noise_sigma > 0.0, "apply_noise: sigma must be positive");
        double* nz = reinterpret_cast<double*>(base + h.off_noise);
        constexpr uint64_t kNoiseTag = 0x4e4f4953;
        const uint64_t step_seed = splitmix_mix(tc->seed, kNoiseTag + static_cast<uint64_t>(step));
        for (int32_t s = 0; s < B; ++s) {
            if (!dn[s]) continue;
            Stream st(splitmix_mix(step_seed, static_cast<uint64_t>(rank) * B + s));
            for (int64_t k = 3 * b->atom_ptr[s]; k < 3 * b->atom_ptr[s + 1]; ++k) nz[k] = st.gauss(0.0, tc->noise_sigma);
        }
    }
    h.B = B;
    h.N = static_cast<int32_t>(N);
    h.me = me, h.mf = mf;
    h.nslots = nslots;
    h.lambda_e = tc ? tc->lambda_energy : 1.0;
    h.lambda_f = tc ? tc->lambda_force : 1.0;
    h.workers = 1;
    h.n_large = 0;
    for (int32_t s = 0; s < B; ++s) {  // samples counted by k_cell_count: all but the small non-periodic ones
        bool periodic = false;
        if (b->cell)
            for (int k = 0; k < 9; ++k) periodic |= b->cell[9 * static_cast<int64_t>(s) + k] != 0.0;
        h.n_large += (b->atom_ptr[s + 1] - b->atom_ptr[s] > kSmallAtoms || periodic) ? 1 : 0;
    }
    std::memcpy(base, &h, sizeof(StepHeader));
    // host mirror
    c.B = B, c.N = N, c.me = me, c.mf = mf, c.n_large = h.n_large;
    c.h_atom_ptr.assign(b->atom_ptr, b->atom_ptr + B + 1);
    c.h_Z.assign(b->atomic_numbers, b->atomic_numbers + N);
    c.h_dsidx.assign(ds, ds + B);
    c.h_emask.assign(em, em + B);
    c.h_fmask.assign(fm, fm + B);
    return off;
}

void collect_step_times(Ctx& c, bool wait_all);
// Step timing: begin / end record a ring slot's event pair on the ctx stream;
// collect_step_times adds the completed intervals in submission order.
int begin_step_events(Ctx& c) {
    if (static_cast<int>(c.ring_pending.size()) == Ctx::kStepRing) {  // ring full: drain the oldest
        CK(cudaEventSynchronize(c.step_ev[c.ring_pending.front()][1]));
        collect_step_times(c, false);
    }
    const int slot = c.ring_next;
    c.ring_next = (c.ring_next + 1) % Ctx::kStepRing;
    CK(cudaEventRecord(c.step_ev[slot][0], c.stream));
    return slot;
}
void end_step_events(Ctx& c, int slot) {
    CK(cudaEventRecord(c.step_ev[slot][1], c.stream));
    c.ring_pending.push_back(slot);
    c.last_slot = slot;
}
void collect_step_times(Ctx& c, bool wait_all) {
    size_t k = 0;
    for (; k < c.ring_pending.size(); ++k) {
        const int slot = c.ring_pending[k];
        if (wait_all) CK(cudaEventSynchronize(c.step_ev[slot][1]));
        else if (cudaEventQuery(c.step_ev[slot][1]) != cudaSuccess) break;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c.step_ev[slot][0], c.step_ev[slot][1]));
        c.step_ms_total += ms;
        ++c.step_count;
        if (c.comm && slot == c.last_slot && c.ring_pending.size() == k + 1) {
            // this rank's own work before the allreduce of the last step (coll_ev is one
            // event recorded by every step's graph: valid for the newest step only)
            float cm = 0.f;
            CK(cudaEventElapsedTime(&cm, c.step_ev[slot][0], c.coll_ev));
            c.compute_ms_last = cm;
        }
    }
    c.ring_pending.erase(c.ring_pending.begin(), c.ring_pending.begin() + static_cast<std::ptrdiff_t>(k));
    (void)cudaGetLastError();  // a cudaEventQuery "not ready" is not an error
}

StepHeader read_header(Ctx& c) {
    CK(cudaMemcpyAsync(c.h_result, c.d_stage.p, sizeof(StepHeader), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    collect_kernel_times(c);
    collect_step_times(c, true);  // device time of the steps so far: upload -> optimizer
    return *c.h_result;
}

// First guess of the directed-pair capacity; overflow regrows it exactly.
int64_t edge_guess(int64_t N) { return 32 * N; }

// Runs the neighbour list, regrowing the edge capacity until it fits.
void run_nlist(Ctx& c) {
    for (int attempt = 0;; ++attempt) {
        c.slot_cursor = 0;
        c.ops->prep(c);  // the per-sample counts and the row offsets live in k_prep
        c.ops->nlist(c);
        const StepHeader h = read_header(c);
        if (!h.overflow) break;
        require(attempt < 4, "neighbour list capacity regrowth did not converge");
        ensure_capacity(c, c.N, c.B, h.P);
    }
    c.nlist_valid = true;
}

void destroy_graphs(Ctx& c) {
    auto kill = [](cudaGraphExec_t& g) {
        if (g) cudaGraphExecDestroy(g);
        g = nullptr;
    };
    auto& a = c.alt_graphs;
    for (cudaGraphExec_t* g : {&c.g_step, &c.g_opt, &c.g_full[0], &c.g_full[1], &c.g_nl[0], &c.g_nl[1], &c.g_model,
                               &a.g_step, &a.g_opt, &a.g_full[0], &a.g_full[1], &a.g_nl[0], &a.g_nl[1], &a.g_model})
        kill(*g);
}

cudaGraphExec_t capture(Ctx& c, void (*body)(Ctx&)) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
        body(c);
    } catch (...) {
        cudaStreamEndCapture(c.stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    CK(cudaStreamEndCapture(c.stream, &g));
    cudaGraphExec_t ex = nullptr;
    CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphDestroy(g));
    return ex;
}

void step_body(Ctx& c) {
    c.ops->prep(c);
    c.ops->nlist(c);
    c.ops->forward(c, false);
    c.ops->loss(c, true);
    c.ops->backward(c, false);
}

void opt_body(Ctx& c) {
    c.ops->opt(c, make_dev(c), c.opt_G, c.opt_inv_g, c.opt_clip, c.opt_lr, c.opt_decay, c.opt_eps);
}

// The gradient allreduce over the ranks (S/trainer.cpp:319: the worker sum),
// in place on the packed fp32 payload [grads | loss hi/lo | overflow | count].
void allreduce_body(Ctx& c) {
    // external: inside a capture a plain record only orders streams; this one is a
    // real event-record node of the graph (timed against step_ev[0])
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(c.stream, &cs));
    if (cs == cudaStreamCaptureStatusActive) CK(cudaEventRecordWithFlags(c.coll_ev, c.stream, cudaEventRecordExternal));
    else CK(cudaEventRecord(c.coll_ev, c.stream));
    nccl_check(nccl().all_reduce(c.grads.p, c.grads.p, static_cast<size_t>(c.NP + 4), ncclFloat32, ncclSum, c.comm,
                                 c.stream),
               "ncclAllReduce");
}

// The whole step after its upload as ONE graph: step -> (communicator: event +
// ncclAllReduce, captured) -> optimizer.
void full_body(Ctx& c) {
    step_body(c);
    if (c.comm) allreduce_body(c);
    opt_body(c);
}

// The two halves of a step for neighbour-list pipelining: the batch preparation
// (denoise, labels, neighbour list; independent of the parameters) and the model
// (forward -> loss -> backward -> allreduce -> optimizer).
void nl_body(Ctx& c) {
    c.ops->prep(c);
    c.ops->nlist(c);
}
void model_body(Ctx& c) {
    c.ops->forward(c, false);
    c.ops->loss(c, true);
    c.ops->backward(c, false);
    if (c.comm) allreduce_body(c);
    opt_body(c);
}

void launch_step(Ctx& c) {
    const int64_t l0 = c.launches;
    if (c.use_graph && !c.profile) {
        // one graph: the optimizer's cooperative launch follows grad_reduce (or the
        // captured allreduce) with programmatic serialization like every other kernel
        if (c.graph_dirty) destroy_graphs(c), c.graph_dirty = false;
        const int variant = c.n_large > 0 ? 1 : 0;
        cudaGraphExec_t& g = c.g_full[variant];
        if (!g) {
            c.slot_cursor = 0;
            c.omit_cell_count = variant == 0;
            try {
                g = capture(c, full_body);
            } catch (...) {
                c.omit_cell_count = false;
                throw;
            }
            c.omit_cell_count = false;
            c.graph_launches = c.launches - l0;
        }
        CK(cudaGraphLaunch(g, c.stream));
        c.last_step_launches = c.graph_launches;
        return;
    }
    if (c.use_graph) {
        if (c.graph_dirty || !c.g_step) {
            destroy_graphs(c);
            c.slot_cursor = 0;
            c.g_step = capture(c, step_body);
            c.g_opt = capture(c, opt_body);
            c.graph_dirty = false;
            c.graph_launches = c.launches - l0;
        }
        CK(cudaGraphLaunch(c.g_step, c.stream));
    } else {
        c.slot_cursor = 0;
        step_body(c);
    }
    if (c.comm) allreduce_body(c);  // profiling pass: between the two graphs
    if (c.use_graph) CK(cudaGraphLaunch(c.g_opt, c.stream));
    else opt_body(c);
    c.last_step_launches = c.use_graph ? c.graph_launches : c.launches - l0;
}

// clear_poison: a rerun of a pipelined (chain) step; every attempt starts with
// the in-flight poison cleared (an overflowing attempt sets it again).
StepHeader run_train_step(Ctx& c, const void* src, size_t bytes, cudaMemcpyKind kind, bool sync = true,
                          bool clear_poison = false) {
    c.grads_in_acc = false;
    for (int attempt = 0;; ++attempt) {
        ensure_capacity(c, c.N, c.B, edge_guess(c.N));
        if (bytes > c.d_stage.bytes) ensure_stage(c, bytes);
        if (clear_poison) CK(cudaMemsetAsync(c.anomaly.as<unsigned int>() + 8, 0, sizeof(unsigned int), c.stream));
        const int ts = begin_step_events(c);
        CK(cudaMemcpyAsync(c.d_stage.p, src, bytes, kind, c.stream));
        launch_step(c);
        end_step_events(c, ts);
        if (!sync) return StepHeader{};
        const StepHeader h = read_header(c);
        if (h.status != 2) {
            // the optimizer in the step graph already rewrote the parameters: the
            // forward cache and the loss gradient belong to the old ones
            c.batch_valid = c.nlist_valid = true;
            c.fwd_valid = c.loss_valid = false;
            return h;
        }
        require(attempt < 4, "edge capacity regrowth did not converge");
        ensure_capacity(c, c.N, c.B, h.overflow ? h.P : 0);
    }
}

// Upload + step graph without the optimizer (one simulated worker); regrows
// the edge capacity and reruns on overflow. Returns the header after the pass.
StepHeader run_pass(Ctx& c, const void* src, size_t bytes, cudaMemcpyKind kind) {
    c.grads_in_acc = false;
    for (int attempt = 0;; ++attempt) {
        ensure_capacity(c, c.N, c.B, edge_guess(c.N));
        if (bytes > c.d_stage.bytes) ensure_stage(c, bytes);
        CK(cudaMemcpyAsync(c.d_stage.p, src, bytes, kind, c.stream));
        if (c.use_graph) {
            if (c.graph_dirty || !c.g_step) {
                destroy_graphs(c);
                c.slot_cursor = 0;
                const int64_t l0 = c.launches;
                c.g_step = capture(c, step_body);
                c.g_opt = capture(c, opt_body);
                c.graph_dirty = false;
                c.graph_launches = c.launches - l0;
            }
            CK(cudaGraphLaunch(c.g_step, c.stream));
        } else {
            c.slot_cursor = 0;
            step_body(c);
        }
        const StepHeader h = read_header(c);
        if (!h.overflow) return h;
        require(attempt < 4, "edge capacity regrowth did not converge");
        ensure_capacity(c, c.N, c.B, h.P);
    }
}

template <class T>
std::vector<T> d2h(Ctx& c, const void* src, size_t count) {
    std::vector<T> out(count);
    if (count) CK(cudaMemcpyAsync(out.data(), src, sizeof(T) * count, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return out;
}

void require_batch(Ctx& c) { require(c.batch_valid, "no batch: call lamm_batch_set first"); }

void ensure_forward(Ctx& c) {
    require_batch(c);
    if (!c.nlist_valid) run_nlist(c);
    if (!c.fwd_valid) {
        c.slot_cursor = 0;
        c.ops->forward(c, true);
        read_header(c);
        c.fwd_valid = true;
    }
}

}  // namespace lamm_b200

using namespace lamm_b200;

// =================================================================== C ABI ==
LAMM_API int lamm_ctx_create(int device, const lamm_model_config* cfg, lamm_ctx** out) {
    return lamm_guard([&] {
        require(cfg && out, "ctx_create: null argument");
        require(cfg->hidden >= 1 && cfg->layers >= 0 && cfg->rbf >= 2 && cfg->cutoff > 0.0 && cfg->heads >= 1,
                "model: invalid config");
        require(cfg->layers >= 1 && cfg->layers <= kMaxLayers, "model: device path supports 1..8 layers");
        require(cfg->heads <= kMaxHeads, "model: device path supports at most 16 heads");
        const Ops* ops = select_ops(cfg->hidden, cfg->rbf);
        require(ops != nullptr, "model: (hidden, rbf) must be one of (128, 8|16), (64, 8|16), (32, 8|16)");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "ctx_create: no such CUDA device");
        auto* c = new lamm_ctx();
        try {
            c->device = device;
            CK(cudaSetDevice(device));
            CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->cfg = *cfg;
            c->H = cfg->hidden, c->L = cfg->layers, c->K = cfg->rbf, c->D = cfg->heads;
            c->NP = lamm_param_count(cfg);
            CK(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device));
            c->ops = ops;
            alloc_param_state(*c);
            c->ops->setup(*c);
            CK(cudaMallocHost(reinterpret_cast<void**>(&c->h_result), sizeof(StepHeader)));
            ensure_stage(*c, 1 << 20);
            for (auto& e : c->ev) CK(cudaEventCreate(&e));
            for (auto& pr : c->step_ev)
                for (auto& e : pr) CK(cudaEventCreate(&e));
            CK(cudaEventCreate(&c->coll_ev));
            ensure_capacity(*c, 1024, 64, 4096);
            // empty reference table buffers so the device pointers are valid
            bool ch = false;
            for (const char* n : {"rho", "rho_has", "tmean", "tstd", "tfstd", "thas"}) ensure_buf(*c, n, 256, ch);
        } catch (...) {
            lamm_ctx_destroy(c);
            throw;
        }
        *out = c;
    });
}

LAMM_API void lamm_ctx_destroy(lamm_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    destroy_graphs(*c);
    if (c->comm) nccl().comm_destroy(c->comm);
    for (auto& kv : c->bufs)
        if (kv.second.p) cudaFree(kv.second.p);
    for (auto& s : c->staged)
        if (s.blob.p) cudaFree(s.blob.p);
    for (Buf* b : {&c->p64, &c->v64, &c->g64, &c->p32, &c->tanh_emb, &c->grads, &c->block_scratch, &c->d_stage,
                   &c->anomaly, &c->flush, &c->wpack})
        if (b->p) cudaFree(b->p);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->h_result) cudaFreeHost(c->h_result);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream), cudaStreamDestroy(c->copy_stream);
    for (auto& f : c->ring) {
        if (f.inbox.p) cudaFree(f.inbox.p);
        if (f.uploaded) cudaEventDestroy(f.uploaded);
        if (f.blob) cudaFreeHost(f.blob);
        if (f.result) cudaFreeHost(f.result);
        if (f.done) cudaEventDestroy(f.done);
        if (f.nl_done) cudaEventDestroy(f.nl_done);
    }
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& pr : c->step_ev)
        for (auto& e : pr)
            if (e) cudaEventDestroy(e);
    if (c->coll_ev) cudaEventDestroy(c->coll_ev);
    if (c->side) cudaStreamSynchronize(c->side), cudaStreamDestroy(c->side);
    for (cudaEvent_t e : {c->ev_prev, c->ev_nl})
        if (e) cudaEventDestroy(e);
    if (c->d_stage_alt.p) cudaFree(c->d_stage_alt.p);
    for (auto& s : c->slots) {
        if (s.a) cudaEventDestroy(s.a);
        if (s.b) cudaEventDestroy(s.b);
    }
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

LAMM_API int lamm_ctx_set_option(lamm_ctx* c, const char* name, int64_t value) {
    return lamm_guard([&] {
        require(c && name, "set_option: null argument");
        const std::string n(name);
        if (n == "graph") c->use_graph = value != 0;
        else if (n == "profile") c->profile = value != 0;
        else if (n == "pdl") c->pdl = value != 0;
        else if (n == "rank_local") c->rank_local = value != 0;
        else if (n == "export_fp64") {
            c->export64 = value != 0;
            require_no_chain(*c);
        CK(cudaSetDevice(c->device));
            ensure_capacity(*c, 0, 0, 0);
            bool ch = false;
            if (c->export64) {
                ensure_buf(*c, "dist64", 8 * c->Pcap, ch);
                ensure_buf(*c, "unit64", 24 * c->Pcap, ch);
            }
            c->nlist_valid = false;
        } else throw InputErr("set_option: unknown option " + n);
        c->graph_dirty = true;
    });
}

LAMM_API int lamm_params_set(lamm_ctx* c, const double* flat, size_t n) {
    return lamm_guard([&] {
        require(c && flat && static_cast<int64_t>(n) == c->NP, "params_set: size mismatch");
        require_no_chain(*c, true);
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpyAsync(c->p64.p, flat, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        Dev d = make_dev(*c);
        k_params_cast<<<c->grid_opt, 256, 0, c->stream>>>(d);
        CK(cudaGetLastError());
        c->ops->pack(*c);
        CK(cudaStreamSynchronize(c->stream));
        c->fwd_valid = c->loss_valid = false;
    });
}

LAMM_API int lamm_params_get(lamm_ctx* c, double* flat, size_t n) {
    return lamm_guard([&] {
        require(c && flat && static_cast<int64_t>(n) == c->NP, "params_get: size mismatch");
        require_no_chain(*c, true);
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpyAsync(flat, c->p64.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

LAMM_API int lamm_rms_state_set(lamm_ctx* c, const double* flat, size_t n) {
    return lamm_guard([&] {
        require(c && flat && static_cast<int64_t>(n) == c->NP, "rms_state_set: size mismatch");
        require_no_chain(*c, true);
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpyAsync(c->v64.p, flat, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

LAMM_API int lamm_rms_state_get(lamm_ctx* c, double* flat, size_t n) {
    return lamm_guard([&] {
        require(c && flat && static_cast<int64_t>(n) == c->NP, "rms_state_get: size mismatch");
        require_no_chain(*c, true);
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpyAsync(flat, c->v64.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

LAMM_API int lamm_ref_table_set(lamm_ctx* c, const lamm_ref_table* t) {
    return lamm_guard([&] {
        require(c != nullptr, "ref_table_set: null ctx");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        if (!t) {
            c->use_table = false;
            c->ntab = 0;
            c->graph_dirty = true;
            return;
        }
        require(t->n_tables >= 1 && t->rho && t->rho_has && t->energy_mean && t->energy_std && t->force_std &&
                    t->has_energy_stats,
                "ref_table_set: incomplete table");
        const int n = t->n_tables;
        bool ch = false;
        ensure_buf(*c, "rho", 8 * 119 * n, ch);
        ensure_buf(*c, "rho_has", 119 * n, ch);
        ensure_buf(*c, "tmean", 8 * n, ch);
        ensure_buf(*c, "tstd", 8 * n, ch);
        ensure_buf(*c, "tfstd", 8 * n, ch);
        ensure_buf(*c, "thas", n, ch);
        auto up = [&](const char* name, const void* src, size_t bytes) {
            CK(cudaMemcpyAsync(buf(*c, name).p, src, bytes, cudaMemcpyHostToDevice, c->stream));
        };
        up("rho", t->rho, 8 * 119 * n);
        up("rho_has", t->rho_has, 119 * n);
        up("tmean", t->energy_mean, 8 * n);
        up("tstd", t->energy_std, 8 * n);
        up("tfstd", t->force_std, 8 * n);
        up("thas", t->has_energy_stats, n);
        CK(cudaStreamSynchronize(c->stream));
        c->h_thas.assign(t->has_energy_stats, t->has_energy_stats + n);
        c->use_table = true;
        c->ntab = n;
        c->graph_dirty = true;
    });
}

LAMM_API int lamm_batch_set(lamm_ctx* c, const lamm_batch_view* b) {
    return lamm_guard([&] {
        require(c != nullptr, "batch_set: null ctx");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        validate_batch(*c, b);
        const size_t bytes = pack_batch(*c, b, false, nullptr, 0, 0);
        ensure_capacity(*c, c->N, c->B, edge_guess(c->N));
        CK(cudaMemcpyAsync(c->d_stage.p, c->h_stage, bytes, cudaMemcpyHostToDevice, c->stream));
        c->slot_cursor = 0;
        c->ops->prep(*c);
        read_header(*c);
        c->batch_valid = true;
        c->nlist_valid = c->fwd_valid = c->loss_valid = false;
    });
}

LAMM_API int lamm_labels_get(lamm_ctx* c, double* energy, double* forces) {
    return lamm_guard([&] {
        require(c != nullptr, "labels_get: null ctx");
        require_batch(*c);
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        if (energy) CK(cudaMemcpyAsync(energy, buf(*c, "En").p, 8 * c->B, cudaMemcpyDeviceToHost, c->stream));
        if (forces) CK(cudaMemcpyAsync(forces, buf(*c, "Fn").p, 24 * c->N, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

LAMM_API int lamm_neighbor_list(lamm_ctx* c, int64_t* n_pairs) {
    return lamm_guard([&] {
        require(c != nullptr, "neighbor_list: null ctx");
        require_batch(*c);
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        if (!c->nlist_valid) run_nlist(*c);
        const StepHeader h = read_header(*c);
        if (n_pairs) *n_pairs = h.P;
    });
}

LAMM_API int lamm_neighbor_list_copy(lamm_ctx* c, int64_t* sample_pair_ptr, int32_t* oi, int32_t* oj, double* dist,
                                     double* unit) {
    return lamm_guard([&] {
        require(c != nullptr, "neighbor_list_copy: null ctx");
        require_batch(*c);
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        if (!c->nlist_valid) run_nlist(*c);
        const StepHeader h = read_header(*c);
        const int64_t P = h.P;
        const auto rp = d2h<int32_t>(*c, buf(*c, "row_ptr").p, c->N + 1);
        const auto col = d2h<int32_t>(*c, buf(*c, "col").p, P);
        for (int32_t s = 0; s < c->B; ++s) {
            const int64_t lo = c->h_atom_ptr[s], hi = c->h_atom_ptr[s + 1];
            if (sample_pair_ptr) sample_pair_ptr[s] = rp[lo];
            for (int64_t i = lo; i < hi; ++i)
                for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
                    if (oi) oi[p] = static_cast<int32_t>(i - lo);
                    if (oj) oj[p] = static_cast<int32_t>(col[p] - lo);
                }
        }
        if (sample_pair_ptr) sample_pair_ptr[c->B] = P;
        if (dist || unit) {
            require(c->export64, "neighbor_list_copy: set option export_fp64 for fp64 distances");
            if (dist) CK(cudaMemcpyAsync(dist, buf(*c, "dist64").p, 8 * P, cudaMemcpyDeviceToHost, c->stream));
            if (unit) CK(cudaMemcpyAsync(unit, buf(*c, "unit64").p, 24 * P, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
    });
}

namespace lamm_b200 {
// [N][D][3] (device) -> per-sample (d*n+j)*3+c (reference Prediction layout)
void to_ref_layout(Ctx& c, const float* src, double* dst) {
    const int D = c.D;
    for (int32_t s = 0; s < c.B; ++s) {
        const int64_t lo = c.h_atom_ptr[s], n = c.h_atom_ptr[s + 1] - lo;
        double* o = dst + 3 * D * lo;
        for (int64_t j = 0; j < n; ++j)
            for (int d = 0; d < D; ++d)
                for (int x = 0; x < 3; ++x) o[(d * n + j) * 3 + x] = src[((lo + j) * D + d) * 3 + x];
    }
}
void from_ref_layout(Ctx& c, const double* src, float* dst) {
    const int D = c.D;
    for (int32_t s = 0; s < c.B; ++s) {
        const int64_t lo = c.h_atom_ptr[s], n = c.h_atom_ptr[s + 1] - lo;
        const double* in = src + 3 * D * lo;
        for (int64_t j = 0; j < n; ++j)
            for (int d = 0; d < D; ++d)
                for (int x = 0; x < 3; ++x) dst[((lo + j) * D + d) * 3 + x] = static_cast<float>(in[(d * n + j) * 3 + x]);
    }
}
}  // namespace lamm_b200

LAMM_API int lamm_forward(lamm_ctx* c, double* energy, double* forces) {
    return lamm_guard([&] {
        require(c != nullptr, "forward: null ctx");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        c->fwd_valid = false;
        ensure_forward(*c);
        if (energy) {
            CK(cudaMemcpyAsync(energy, buf(*c, "Epred").p, 8 * c->B * c->D, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
        if (forces) {
            const auto F = d2h<float>(*c, buf(*c, "F").p, 3 * c->N * c->D);
            to_ref_layout(*c, F.data(), forces);
        }
    });
}

LAMM_API int lamm_evaluate(lamm_ctx* c, const lamm_batch_view* b, lamm_eval_result* out) {
    return lamm_guard([&] {
        require(c && b && out, "evaluate: null argument");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        lamm_batch_view v = *b;
        v.denoise = nullptr;  // evaluate() takes the samples as given
        validate_batch(*c, &v);
        const size_t bytes = pack_batch(*c, &v, false, nullptr, 0, 0);
        ensure_capacity(*c, c->N, c->B, edge_guess(c->N));
        CK(cudaMemcpyAsync(c->d_stage.p, c->h_stage, bytes, cudaMemcpyHostToDevice, c->stream));
        c->slot_cursor = 0;
        c->ops->prep(*c);
        read_header(*c);
        c->batch_valid = true;
        c->nlist_valid = c->fwd_valid = c->loss_valid = false;
        ensure_forward(*c);
        launch(*c, "eval", k_eval, c->grid_small, 128, 0, make_dev(*c));
        const StepHeader h = read_header(*c);
        int64_t ne = 0, nf = 0;
        for (int32_t s = 0; s < c->B; ++s) ne += c->h_emask[s] ? 1 : 0, nf += c->h_fmask[s] ? 1 : 0;
        out->energy_count = ne;
        out->force_count = nf;
        out->energy_mae = ne > 0 ? 1000.0 * h.loss_energy / static_cast<double>(ne) : std::nan("");
        out->force_mae = nf > 0 ? 1000.0 * h.loss_force / static_cast<double>(nf) : std::nan("");
    });
}

LAMM_API int lamm_forward_cache_get(lamm_ctx* c, int which, int layer, double* out) {
    return lamm_guard([&] {
        require(c && out, "forward_cache_get: null argument");
        require_batch(*c);
        require(c->fwd_valid, "forward_cache_get: run lamm_forward first");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        const int H = c->H;
        std::vector<float> v;
        if (which == 0) {
            require(layer >= 0 && layer <= c->L, "forward_cache_get: layer out of range");
            if (layer == 0) {
                const auto emb = d2h<float>(*c, c->p32.p, static_cast<size_t>(kMaxZ) * H);
                v.resize(static_cast<size_t>(c->N) * H);
                for (int64_t i = 0; i < c->N; ++i)
                    std::copy_n(emb.begin() + static_cast<int64_t>(c->h_Z[i] - 1) * H, H, v.begin() + i * H);
            } else {
                v = d2h<float>(*c, buf(*c, "h" + std::to_string(layer)).p, static_cast<size_t>(c->N) * H);
            }
        } else {
            require(layer >= 0 && layer < c->L, "forward_cache_get: layer out of range");
            v = d2h<float>(*c, buf(*c, "mu" + std::to_string(layer)).p, static_cast<size_t>(c->N) * H);
        }
        for (size_t k = 0; k < v.size(); ++k) out[k] = v[k];
    });
}

LAMM_API int lamm_loss_grad(lamm_ctx* c, const lamm_loss_config* cfg, lamm_loss_breakdown* out, double* g_energy,
                            double* g_forces) {
    return lamm_guard([&] {
        require(c != nullptr, "loss_grad: null ctx");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        const double le = cfg ? cfg->lambda_energy : 1.0, lf = cfg ? cfg->lambda_force : 1.0;
        require(le >= 0.0 && lf >= 0.0, "masked_loss: lambdas must be non-negative");
        ensure_forward(*c);
        StepHeader* hd = reinterpret_cast<StepHeader*>(c->h_stage);  // staged header copy
        hd->lambda_e = le, hd->lambda_f = lf;
        CK(cudaMemcpyAsync(c->d_stage.as<char>() + offsetof(StepHeader, lambda_e), &hd->lambda_e, 16,
                           cudaMemcpyHostToDevice, c->stream));
        c->slot_cursor = 0;
        c->ops->loss(*c, false);
        const StepHeader h = read_header(*c);
        if (out) {
            out->total = h.loss_total;
            out->energy_term = h.loss_energy;
            out->force_term = h.loss_force;
            out->energy_labeled = c->me;
            out->force_labeled = c->mf;
            out->energy_empty = c->me == 0;
            out->force_empty = c->mf == 0;
        }
        if (g_energy) {
            const auto ge = d2h<float>(*c, buf(*c, "gE").p, static_cast<size_t>(c->B) * c->D);
            for (size_t k = 0; k < ge.size(); ++k) g_energy[k] = ge[k];
        }
        if (g_forces) {
            const auto gf = d2h<float>(*c, buf(*c, "gF").p, 3 * c->N * c->D);
            to_ref_layout(*c, gf.data(), g_forces);
        }
        c->loss_valid = true;
    });
}

LAMM_API int lamm_backward(lamm_ctx* c, const double* up_energy, const double* up_forces, double* grads_accum) {
    return lamm_guard([&] {
        require(c != nullptr, "backward: null ctx");
        c->grads_in_acc = false;
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        ensure_forward(*c);
        const bool general = up_energy || up_forces;
        if (general) {
            std::vector<float> ge(static_cast<size_t>(c->B) * c->D, 0.f), gf(3 * c->N * c->D, 0.f);
            if (up_energy)
                for (size_t k = 0; k < ge.size(); ++k) ge[k] = static_cast<float>(up_energy[k]);
            if (up_forces) from_ref_layout(*c, up_forces, gf.data());
            CK(cudaMemcpyAsync(buf(*c, "gE").p, ge.data(), 4 * ge.size(), cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(buf(*c, "gF").p, gf.data(), 4 * gf.size(), cudaMemcpyHostToDevice, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        } else {
            require(c->loss_valid, "backward: no upstream gradient (pass one or call lamm_loss_grad)");
        }
        c->slot_cursor = 0;
        c->ops->backward(*c, general);
        read_header(*c);
        if (grads_accum) {
            const auto g = d2h<float>(*c, c->grads.p, c->NP);
            for (int64_t k = 0; k < c->NP; ++k) grads_accum[k] += g[k];
        }
    });
}

LAMM_API int lamm_grads_get(lamm_ctx* c, double* flat, size_t n) {
    return lamm_guard([&] {
        require(c && flat && static_cast<int64_t>(n) == c->NP, "grads_get: size mismatch");
        require_no_chain(*c, true);
        CK(cudaSetDevice(c->device));
        if (c->grads_in_acc) {  // simulated workers: the fp64 worker sum the optimizer consumed
            CK(cudaMemcpyAsync(flat, c->g64.p, sizeof(double) * c->NP, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            return;
        }
        const auto g = d2h<float>(*c, c->grads.p, c->NP);
        for (int64_t k = 0; k < c->NP; ++k) flat[k] = g[k];
    });
}

LAMM_API int lamm_comm_unique_id(void* out128) {
    return lamm_guard([&] {
        require(out128 != nullptr, "comm_unique_id: null output");
        if (!nccl().ok) throw NcclErr("libnccl.so.2 could not be loaded");
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof(id));
    });
}

LAMM_API int lamm_comm_init(lamm_ctx* c, int nranks, int rank, const void* id128) {
    return lamm_guard([&] {
        require(c && id128, "comm_init: null argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: bad rank layout");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        require(c->comm == nullptr, "comm_init: the context already has a communicator");
        // a real communicator even for one rank: the step then runs the same
        // captured allreduce as every rank of a multi-GPU job
        if (!nccl().ok) throw NcclErr("libnccl.so.2 could not be loaded");
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        nccl_check(nccl().comm_init_rank(&c->comm, nranks, id, rank), "ncclCommInitRank");
        c->nranks = nranks, c->rank = rank;
        c->graph_dirty = true;
    });
}

namespace lamm_b200 {
// simulated: lamm_train_step_workers runs every worker on this ctx and sums them itself
void apply_train_config(Ctx& c, const lamm_train_config* tc, int32_t workers, int32_t rank, bool simulated = false) {
    require(workers >= 1 && rank >= 0 && rank < workers, "train_step: bad worker layout");
    if (c.comm) {
        require(workers == c.nranks && rank == c.rank, "train_step: workers/rank must match the communicator");
    } else if (workers > 1 && !simulated) {
        // without a communicator a workers > 1 step would apply this rank's gradient
        // alone (scaled 1/G) - not the reference step (S/trainer.cpp:319-326)
        require(c.rank_local,
                "train_step: workers > 1 needs a communicator (lamm_comm_init) or lamm_train_step_workers; "
                "set option rank_local to run one rank's share on its own");
    }
    require(tc->learning_rate > 0.0, "train: learning_rate must be positive");
    require(tc->clip_norm >= 0.0, "train: clip_norm must be >= 0");
    require(tc->rms_decay >= 0.0 && tc->rms_decay < 1.0, "train: rms_decay must be in [0, 1)");
    require(tc->rms_epsilon > 0.0, "train: rms_epsilon must be positive");
    require(tc->lambda_energy >= 0.0 && tc->lambda_force >= 0.0, "train: lambdas must be >= 0");
    if (c.denoise_scheme != (tc->noise_scheme ? 1 : 0)) {
        c.denoise_scheme = tc->noise_scheme ? 1 : 0;
        c.graph_dirty = true;
    }
    const double inv_g = 1.0 / static_cast<double>(workers);
    if (c.opt_inv_g != inv_g || c.opt_lr != tc->learning_rate || c.opt_decay != tc->rms_decay ||
        c.opt_eps != tc->rms_epsilon || c.opt_clip != tc->clip_norm || c.opt_G != workers) {
        c.opt_inv_g = inv_g, c.opt_lr = tc->learning_rate, c.opt_decay = tc->rms_decay;
        c.opt_eps = tc->rms_epsilon, c.opt_clip = tc->clip_norm, c.opt_G = workers;
        c.graph_dirty = true;
    }
}

void fill_result(Ctx& c, const StepHeader& h, lamm_step_result* res) {
    if (!res) return;
    res->loss = h.global_loss;
    res->grad_norm = h.grad_norm;
    res->local.total = h.loss_total;
    res->local.energy_term = h.loss_energy;
    res->local.force_term = h.loss_force;
    res->local.energy_labeled = c.me;
    res->local.force_labeled = c.mf;
    res->local.energy_empty = c.me == 0;
    res->local.force_empty = c.mf == 0;
    res->n_atoms = c.N;
    res->n_edges = h.P;
    res->status = h.status == 1 ? LAMM_ENONFINITE : LAMM_OK;
    res->retries = 0;
    res->h2d_bytes = c.last_h2d;
    res->d2h_bytes = static_cast<int64_t>(sizeof(StepHeader));
}
// Enqueues one pipelined step: upload of the slot's pinned blob, the step and
// optimizer graphs, and the read-back of its header into the slot's pinned
// result, then the slot's completion event. Capacity growth or a graph
// recapture first drains the stream (nothing in flight is reallocated).
void launch_nl(Ctx& c, cudaStream_t stream);
void launch_model(Ctx& c);

// The side stream of the batch preparation at the LOWEST priority: its blocks take
// SMs only when the model's kernels leave them idle, never ahead of them (measured:
// the same step time as the default priority; the highest priority costs 4 %).
void create_side_stream(Ctx& c) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking, lo));
}

void enqueue_chained(Ctx& c, Ctx::Inflight& f) {
    c.B = f.B, c.N = f.N, c.me = f.me, c.mf = f.mf, c.n_large = f.n_large;
    apply_train_config(c, &f.tc, f.workers, f.rank);
    // graphs on: the step's batch preparation runs on the side stream into the batch-
    // state parity the in-flight step does not use, overlapping that step's model
    const bool pipe = c.use_graph && !c.profile;
    if (pipe && !c.side) {
        create_side_stream(c);
        CK(cudaEventCreateWithFlags(&c.ev_prev, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c.ev_nl, cudaEventDisableTiming));
    }
    if (c.graph_dirty || f.N > c.Ncap || f.B > c.Bcap || edge_guess(f.N) > c.Pcap || f.bytes > c.d_stage.bytes ||
        (pipe && (!c.pipe_alloc || f.bytes > c.d_stage_alt.bytes))) {
        CK(cudaStreamSynchronize(c.stream));
        if (c.side) CK(cudaStreamSynchronize(c.side));
    }
    c.pipe_valid = false;
    if (pipe) c.pipe_alloc = true;
    ensure_capacity(c, f.N, f.B, edge_guess(f.N));
    ensure_stage(c, f.bytes);
    // the upload runs on the copy stream while the previous step computes; the
    // step's stream waits for it and moves the blob into the staging buffer (D2D)
    if (!c.copy_stream) CK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    if (!f.uploaded) CK(cudaEventCreateWithFlags(&f.uploaded, cudaEventDisableTiming));
    if (f.inbox.bytes < f.bytes) {
        if (f.inbox.p) CK(cudaFree(f.inbox.p));
        CK(cudaMalloc(&f.inbox.p, f.cap));
        f.inbox.bytes = f.cap;
    }
    CK(cudaMemcpyAsync(f.inbox.p, f.blob, f.bytes, cudaMemcpyHostToDevice, c.copy_stream));
    CK(cudaEventRecord(f.uploaded, c.copy_stream));
    if (!pipe) {
        CK(cudaStreamWaitEvent(c.stream, f.uploaded, 0));
        CK(cudaMemcpyAsync(c.d_stage.p, f.inbox.p, f.bytes, cudaMemcpyDeviceToDevice, c.stream));
        launch_step(c);
    } else {
        if (c.graph_dirty) destroy_graphs(c), c.graph_dirty = false;
        if (!f.nl_done) CK(cudaEventCreateWithFlags(&f.nl_done, cudaEventDisableTiming));
        // the other parity's last user is the step before the in-flight one, already
        // waited for (at most two in flight); the side stream keeps the order of the
        // batch preparations
        swap_parity(c);  // (the ring alternates parities; a failure below leaves it swapped: still consistent)
        CK(cudaStreamWaitEvent(c.side, f.uploaded, 0));
        CK(cudaMemcpyAsync(c.d_stage.p, f.inbox.p, f.bytes, cudaMemcpyDeviceToDevice, c.side));
        launch_nl(c, c.side);
        CK(cudaEventRecord(f.nl_done, c.side));
        CK(cudaStreamWaitEvent(c.stream, f.nl_done, 0));
        launch_model(c);
        c.last_step_launches = c.graph_launches + (c.n_large > 0 ? 3 : 2);
    }
    CK(cudaMemcpyAsync(f.result, c.d_stage.p, sizeof(StepHeader), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaEventRecord(f.done, c.stream));
}

}  // namespace lamm_b200

LAMM_API int lamm_stage(lamm_ctx* c, const lamm_batch_view* b, const lamm_train_config* tc, int64_t step,
                        int32_t workers, int32_t rank, int32_t slot) {
    return lamm_guard([&] {
        require(c && b && tc, "stage: null argument");
        require(slot >= 0 && slot < 1024, "stage: slot out of range");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        validate_batch(*c, b);
        apply_train_config(*c, tc, workers, rank);
        const size_t bytes = pack_batch(*c, b, true, tc, step, rank);
        if (static_cast<size_t>(slot) >= c->staged.size()) c->staged.resize(slot + 1);
        auto& s = c->staged[slot];
        if (s.blob.bytes < bytes) {
            if (s.blob.p) CK(cudaFree(s.blob.p));
            CK(cudaMalloc(&s.blob.p, bytes));
            s.blob.bytes = bytes;
        }
        CK(cudaMemcpyAsync(s.blob.p, c->h_stage, bytes, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        s.bytes = bytes, s.B = c->B, s.N = c->N, s.me = c->me, s.mf = c->mf, s.n_large = c->n_large;
        ensure_capacity(*c, c->N, c->B, edge_guess(c->N));
    });
}

LAMM_API int lamm_train_step_staged(lamm_ctx* c, int32_t slot, int32_t sync, lamm_step_result* res) {
    return lamm_guard([&] {
        require(c != nullptr, "train_step_staged: null ctx");
        require(slot >= 0 && static_cast<size_t>(slot) < c->staged.size() && c->staged[slot].bytes > 0,
                "train_step_staged: empty slot");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        auto& s = c->staged[slot];
        c->B = s.B, c->N = s.N, c->me = s.me, c->mf = s.mf, c->n_large = s.n_large;
        c->batch_valid = false;  // the host mirror of per-atom arrays is not kept for staged batches
        const StepHeader h = run_train_step(*c, s.blob.p, s.bytes, cudaMemcpyDeviceToDevice, sync != 0);
        c->last_h2d = 0;
        c->batch_valid = c->nlist_valid = c->fwd_valid = c->loss_valid = false;
        if (!sync) return;
        fill_result(*c, h, res);
        if (h.status == 1) throw NonFinite("non-finite loss or gradient");
    });
}

namespace lamm_b200 {
// The batch-preparation graph (variant: with k_cell_count or not) of the current
// parity on `stream`, captured on first use.
void launch_nl(Ctx& c, cudaStream_t stream) {
    const int v = c.n_large > 0 ? 1 : 0;
    cudaGraphExec_t& g = c.g_nl[v];
    if (!g) {
        c.slot_cursor = 0;
        c.omit_cell_count = v == 0;
        try {
            g = capture(c, nl_body);
        } catch (...) {
            c.omit_cell_count = false;
            throw;
        }
        c.omit_cell_count = false;
    }
    CK(cudaGraphLaunch(g, stream));
}
void launch_model(Ctx& c) {
    if (!c.g_model) {
        const int64_t l0 = c.launches;
        c.slot_cursor = 0;
        c.g_model = capture(c, model_body);
        c.graph_launches = c.launches - l0;
    }
    CK(cudaGraphLaunch(c.g_model, c.stream));
}
}  // namespace lamm_b200

// A staged step whose batch preparation (denoise, labels, neighbour list: k_prep,
// k_cell_count, k_nbr_fill — independent of the parameters) was built ahead, while
// the previous step's model ran, into the other batch-state parity; this call in
// turn builds `next_slot`'s on the side stream during its own model. The step's
// device interval (step_ev) covers its model and the prefetch it overlaps, so the
// summed step times still contain every neighbour list that ran.
LAMM_API int lamm_train_step_staged_next(lamm_ctx* c, int32_t slot, int32_t next_slot, int32_t sync,
                                         lamm_step_result* res) {
    return lamm_guard([&] {
        require(c != nullptr, "train_step_staged_next: null ctx");
        auto ok_slot = [&](int32_t k) {
            return k >= 0 && static_cast<size_t>(k) < c->staged.size() && c->staged[k].bytes > 0;
        };
        require(ok_slot(slot), "train_step_staged_next: empty slot");
        require(next_slot < 0 || ok_slot(next_slot), "train_step_staged_next: empty next slot");
        require(c->oldest_ticket == c->next_ticket, "call while pipelined steps are in flight (lamm_train_step_wait first)");
        require(c->use_graph && !c->profile, "train_step_staged_next: needs graph capture (option graph 1, profile 0)");
        CK(cudaSetDevice(c->device));
        if (!c->side) {
            create_side_stream(*c);
            CK(cudaEventCreateWithFlags(&c->ev_prev, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_nl, cudaEventDisableTiming));
        }
        const auto& s = c->staged[slot];
        const Ctx::Slot* nx = next_slot >= 0 ? &c->staged[next_slot] : nullptr;
        // capacity for both batches before anything is enqueued (growth drains first)
        const int64_t N = std::max<int64_t>(s.N, nx ? nx->N : 0);
        const int64_t B = std::max<int64_t>(s.B, nx ? nx->B : 0);
        const size_t bytes = std::max(s.bytes, nx ? nx->bytes : 0);
        const bool grow = !c->pipe_alloc || N > c->Ncap || B > c->Bcap || edge_guess(N) > c->Pcap ||
                          bytes > c->d_stage.bytes || bytes > c->d_stage_alt.bytes || c->graph_dirty;
        if (grow) {
            CK(cudaStreamSynchronize(c->stream));
            drain_pipe(*c);
            c->pipe_alloc = true;
            ensure_capacity(*c, N, B, edge_guess(N));
            ensure_stage(*c, bytes);
            if (c->graph_dirty) destroy_graphs(*c), c->graph_dirty = false;
        }
        const bool pre = c->pipe_valid && c->pipe_slot == slot;
        if (pre) swap_parity(*c);  // the prefetched batch state becomes the current one
        c->B = s.B, c->N = s.N, c->me = s.me, c->mf = s.mf, c->n_large = s.n_large;
        c->grads_in_acc = false;
        const int ts = begin_step_events(*c);
        if (pre) {
            CK(cudaStreamWaitEvent(c->stream, c->ev_nl, 0));
        } else {
            CK(cudaMemcpyAsync(c->d_stage.p, s.blob.p, s.bytes, cudaMemcpyDeviceToDevice, c->stream));
            launch_nl(*c, c->stream);
        }
        // the other parity is free once everything before this step's model is done
        CK(cudaEventRecord(c->ev_prev, c->stream));
        launch_model(*c);
        c->last_step_launches = c->graph_launches;
        c->pipe_valid = false;
        if (nx) {
            swap_parity(*c);
            c->n_large = nx->n_large;
            try {
                CK(cudaStreamWaitEvent(c->side, c->ev_prev, 0));
                CK(cudaMemcpyAsync(c->d_stage.p, nx->blob.p, nx->bytes, cudaMemcpyDeviceToDevice, c->side));
                launch_nl(*c, c->side);
                CK(cudaEventRecord(c->ev_nl, c->side));
            } catch (...) {  // keep the current step's parity current
                swap_parity(*c);
                c->n_large = s.n_large;
                throw;
            }
            swap_parity(*c);
            c->n_large = s.n_large;
            c->pipe_valid = true, c->pipe_slot = next_slot;
            CK(cudaStreamWaitEvent(c->stream, c->ev_nl, 0));  // the step's interval covers the prefetch
            c->last_step_launches += c->n_large > 0 ? 3 : 2;
        }
        end_step_events(*c, ts);
        c->last_h2d = 0;
        c->batch_valid = c->nlist_valid = c->fwd_valid = c->loss_valid = false;
        if (!sync) return;
        StepHeader h = read_header(*c);
        if (h.status == 2) {  // this batch overflowed the edge capacity: regrow, rerun it unpipelined
            drain_pipe(*c);
            ensure_capacity(*c, c->N, c->B, h.overflow ? h.P : 0);
            h = run_train_step(*c, s.blob.p, s.bytes, cudaMemcpyDeviceToDevice, true);
        }
        fill_result(*c, h, res);
        if (h.status == 1) throw NonFinite("non-finite loss or gradient");
    });
}

LAMM_API int64_t lamm_anomalies(lamm_ctx* c) {
    if (!c) return -1;
    unsigned int v = 0;
    if (cudaMemcpy(&v, c->anomaly.p, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return v;
}

LAMM_API int lamm_flush_l2(lamm_ctx* c, int64_t bytes) {
    return lamm_guard([&] {
        require(c != nullptr && bytes > 0, "flush_l2: bad argument");
        CK(cudaSetDevice(c->device));
        if (c->flush.bytes < static_cast<size_t>(bytes)) {
            if (c->flush.p) CK(cudaFree(c->flush.p));
            CK(cudaMalloc(&c->flush.p, bytes));
            c->flush.bytes = bytes;
        }
        CK(cudaMemsetAsync(c->flush.p, c->flush_flip ^= 1, bytes, c->stream));
    });
}

LAMM_API int lamm_train_step(lamm_ctx* c, const lamm_batch_view* b, const lamm_train_config* tc, int64_t step,
                             int32_t workers, int32_t rank, lamm_step_result* res) {
    return lamm_guard([&] {
        require(c && b && tc, "train_step: null argument");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        validate_batch(*c, b);
        apply_train_config(*c, tc, workers, rank);
        const size_t bytes = pack_batch(*c, b, true, tc, step, rank);
        const StepHeader h = run_train_step(*c, c->h_stage, bytes, cudaMemcpyHostToDevice);
        c->last_h2d = static_cast<int64_t>(bytes);
        fill_result(*c, h, res);
        if (h.status == 1)
            throw NonFinite("non-finite loss or gradient at step " + std::to_string(step));
    });
}


LAMM_API int lamm_train_step_submit(lamm_ctx* c, const lamm_batch_view* b, const lamm_train_config* tc, int64_t step,
                                    int32_t workers, int32_t rank, int64_t* ticket) {
    return lamm_guard([&] {
        require(c && b && tc && ticket, "train_step_submit: null argument");
        require(c->next_ticket - c->oldest_ticket < 2, "train_step_submit: two steps in flight; wait for the oldest");
        CK(cudaSetDevice(c->device));
        validate_batch(*c, b);
        apply_train_config(*c, tc, workers, rank);  // validation (enqueue re-applies it)
        auto& f = c->ring[c->next_ticket & 1];
        if (!f.result) CK(cudaMallocHost(reinterpret_cast<void**>(&f.result), sizeof(StepHeader)));
        if (!f.done) CK(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming));
        // pack into the slot's own pinned blob (its previous step has completed:
        // at most two in flight and this slot's ticket was waited for)
        std::swap(c->h_stage, f.blob);
        std::swap(c->h_stage_cap, f.cap);
        size_t bytes = 0;
        try {
            bytes = pack_batch(*c, b, true, tc, step, rank);
        } catch (...) {
            std::swap(c->h_stage, f.blob);
            std::swap(c->h_stage_cap, f.cap);
            throw;
        }
        std::swap(c->h_stage, f.blob);
        std::swap(c->h_stage_cap, f.cap);
        reinterpret_cast<StepHeader*>(f.blob)->chain = 1;
        f.bytes = bytes, f.B = c->B, f.N = c->N, f.me = c->me, f.mf = c->mf, f.n_large = c->n_large;
        f.step = step, f.workers = workers, f.rank = rank, f.tc = *tc;
        c->batch_valid = c->nlist_valid = c->fwd_valid = c->loss_valid = false;
        enqueue_chained(*c, f);
        *ticket = c->next_ticket++;
    });
}

LAMM_API int lamm_train_step_wait(lamm_ctx* c, int64_t ticket, lamm_step_result* res) {
    return lamm_guard([&] {
        require(c != nullptr, "train_step_wait: null ctx");
        require(ticket == c->oldest_ticket && ticket < c->next_ticket, "train_step_wait: not the oldest ticket in flight");
        CK(cudaSetDevice(c->device));
        auto& f = c->ring[ticket & 1];
        CK(cudaEventSynchronize(f.done));
        if (f.result->status == 2 || f.result->status == 3) {
            // capacity overflow, or skipped behind a failed in-flight step: drain, clear
            // the poison, rerun this step and the later in-flight ones in order
            // (run_train_step regrows capacity until the step fits)
            CK(cudaStreamSynchronize(c->stream));
            if (c->side) CK(cudaStreamSynchronize(c->side));
            CK(cudaMemsetAsync(c->anomaly.as<unsigned int>() + 8, 0, sizeof(unsigned int), c->stream));
            for (int64_t t = ticket; t < c->next_ticket; ++t) {
                auto& g = c->ring[t & 1];
                c->B = g.B, c->N = g.N, c->me = g.me, c->mf = g.mf, c->n_large = g.n_large;
                apply_train_config(*c, &g.tc, g.workers, g.rank);
                *g.result = run_train_step(*c, g.blob, g.bytes, cudaMemcpyHostToDevice, true, true);
                if (g.result->status == 1) {  // later ones stay "skipped" and rerun at their wait
                    for (int64_t u = t + 1; u < c->next_ticket; ++u) c->ring[u & 1].result->status = 3;
                    break;
                }
            }
        }
        const StepHeader h = *f.result;
        c->oldest_ticket = ticket + 1;
        if (h.status == 1 && c->oldest_ticket == c->next_ticket)  // nothing behind it: clear the poison now
            CK(cudaMemsetAsync(c->anomaly.as<unsigned int>() + 8, 0, sizeof(unsigned int), c->stream));
        c->B = f.B, c->N = f.N, c->me = f.me, c->mf = f.mf, c->n_large = f.n_large;
        c->last_h2d = static_cast<int64_t>(f.bytes);
        fill_result(*c, h, res);
        if (h.status == 1) throw NonFinite("non-finite loss or gradient at step " + std::to_string(f.step));
    });
}

LAMM_API int lamm_train_step_workers(lamm_ctx* c, const lamm_batch_view* batches, int32_t workers,
                                     const lamm_train_config* tc, int64_t step, lamm_step_result* res) {
    return lamm_guard([&] {
        require(c && batches && tc, "train_step_workers: null argument");
        require(workers >= 1, "train_step_workers: workers must be >= 1");
        require(c->comm == nullptr, "train_step_workers: simulated workers need a context without a communicator");
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        int64_t atoms = 0, edges = 0;
        for (int32_t g = 0; g < workers; ++g) {  // worker order, like S/trainer.cpp:262
            validate_batch(*c, &batches[g]);
            apply_train_config(*c, tc, workers, g, true);
            const size_t bytes = pack_batch(*c, &batches[g], true, tc, step, g);
            const StepHeader h = run_pass(*c, c->h_stage, bytes, cudaMemcpyHostToDevice);
            atoms += c->N, edges += h.P;
            launch(*c, "grad_accum", k_grad_accum, c->grid_small, 256, 0, make_dev(*c), g == 0 ? 1 : 0);
        }
        Dev d = make_dev(*c);
        d.g64_in = c->g64.as<double>();
        d.g64_loss = 1;
        c->ops->opt(*c, d, workers, 1.0 / static_cast<double>(workers), tc->clip_norm, tc->learning_rate,
                    tc->rms_decay, tc->rms_epsilon);
        const StepHeader h = read_header(*c);
        c->batch_valid = c->nlist_valid = true;  // the last worker's batch stays current
        c->fwd_valid = c->loss_valid = false;    // its parameters changed
        c->grads_in_acc = true;
        c->last_h2d = 0;
        fill_result(*c, h, res);
        if (res) res->n_atoms = atoms, res->n_edges = edges;
        if (h.status == 1)
            throw NonFinite("non-finite loss or gradient at step " + std::to_string(step));
    });
}

LAMM_API int lamm_optimizer_step(lamm_ctx* c, const double* grad_sum, int32_t workers, const lamm_train_config* tc,
                                 double* grad_norm) {
    return lamm_guard([&] {
        require(c && grad_sum && tc, "optimizer_step: null argument");
        require(workers >= 1, "optimizer_step: workers must be >= 1");
        c->grads_in_acc = false;
        require_no_chain(*c);
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpyAsync(c->g64.p, grad_sum, sizeof(double) * c->NP, cudaMemcpyHostToDevice, c->stream));
        Dev d = make_dev(*c);
        d.g64_in = c->g64.as<double>();
        const double inv_g = 1.0 / static_cast<double>(workers);
        c->ops->opt(*c, d, workers, inv_g, tc->clip_norm, tc->learning_rate, tc->rms_decay, tc->rms_epsilon);
        const StepHeader h = read_header(*c);
        if (grad_norm) *grad_norm = h.grad_norm;
        c->fwd_valid = c->loss_valid = false;
        if (h.status == 1) throw NonFinite("non-finite gradient");
    });
}

LAMM_API int lamm_sync(lamm_ctx* c) {
    return lamm_guard([&] {
        require(c != nullptr, "sync: null ctx");
        CK(cudaStreamSynchronize(c->stream));
    });
}

LAMM_API int lamm_event_record(lamm_ctx* c, int slot) {
    return lamm_guard([&] {
        require(c && slot >= 0 && slot < 64, "event_record: bad slot");
        CK(cudaEventRecord(c->ev[slot], c->stream));
    });
}

LAMM_API int lamm_event_elapsed_ms(lamm_ctx* c, int a, int b, float* ms) {
    return lamm_guard([&] {
        require(c && ms && a >= 0 && a < 64 && b >= 0 && b < 64, "event_elapsed: bad slot");
        CK(cudaEventSynchronize(c->ev[b]));
        CK(cudaEventElapsedTime(ms, c->ev[a], c->ev[b]));
    });
}

LAMM_API int lamm_kernel_times(lamm_ctx* c, int max_kernels, const char** names, double* total_ms, int64_t* launches,
                               int* n_kernels) {
    return lamm_guard([&] {
        require(c != nullptr, "kernel_times: null ctx");
        int k = 0;
        for (const auto& kv : c->ktimes) {
            if (k < max_kernels) {
                if (names) names[k] = kv.first.c_str();
                if (total_ms) total_ms[k] = kv.second.first;
                if (launches) launches[k] = kv.second.second;
            }
            ++k;
        }
        if (n_kernels) *n_kernels = k;
    });
}

LAMM_API int lamm_kernel_times_reset(lamm_ctx* c) {
    return lamm_guard([&] {
        require(c != nullptr, "kernel_times_reset: null ctx");
        c->ktimes.clear();
        c->ring_pending.clear();  // intervals not yet collected belong to the old window
        c->step_ms_total = 0.0;
        c->step_count = 0;
    });
}

LAMM_API int lamm_step_times(lamm_ctx* c, double* total_ms, int64_t* steps) {
    return lamm_guard([&] {
        require(c != nullptr, "step_times: null ctx");
        collect_step_times(*c, true);  // steps submitted without a sync included
        if (total_ms) *total_ms = c->step_ms_total;
        if (steps) *steps = c->step_count;
    });
}

LAMM_API int64_t lamm_last_step_launches(lamm_ctx* c) { return c ? c->last_step_launches : -1; }

LAMM_API int lamm_last_step_compute_ms(lamm_ctx* c, double* ms) {
    return lamm_guard([&] {
        require(c && ms, "last_step_compute_ms: null argument");
        require(c->comm != nullptr, "last_step_compute_ms: needs a communicator (lamm_comm_init)");
        *ms = c->compute_ms_last;
    });
}

LAMM_API int lamm_ctx_get_info(lamm_ctx* c, const char* name, int64_t* value) {
    return lamm_guard([&] {
        require(c && name && value, "get_info: null argument");
        const std::string n(name);
        if (n == "grid_edge") *value = c->grid_edge;
        else if (n == "parts_per_cta") *value = kPartsPerCta;
        else if (n == "chunk_edges") *value = kChunk;
        else if (n == "atom_cost") *value = kAtomCost;
        else if (n == "message_groups") *value = kMsgGroups;
        else if (n == "message_block") *value = MessageBody<128, 16, true, false>::kBlock;
        else if (n == "edge_groups") *value = kGroups;
        else if (n == "edge_block") *value = BwdBody<128, 16, true, false>::kBlock;
        else if (n == "force_groups") *value = kForceGroups;
        else if (n == "sm_count") *value = c->nsm;
        else if (n == "edge_capacity") *value = c->Pcap;
        else throw InputErr("get_info: unknown name " + n);
    });
}

LAMM_API int lamm_cell_inverse(const double* cell, double* out) {
    return lamm_guard([&] {
        require(cell && out, "cell_inverse: null argument");
        require(cell_inverse(cell, out), "cell: singular");
    });
}
