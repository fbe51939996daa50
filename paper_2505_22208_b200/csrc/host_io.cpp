// host_io.cpp - the on-disk formats next to the train step:
//
//   LAMMCKPT checkpoints ... S/model.cpp:429-497: magic "LAMMCKPT", u32 version 1,
//                            u32 hidden, layers, rbf, heads, f64 cutoff, then per
//                            tensor (for_each_tensor order) u32 rows, u32 cols and
//                            rows*cols f64, all little-endian. Written and read
//                            bit-exactly like the reference.
//   LAMMRMS1 optimizer state  the RMS accumulator v in the same tensor layout
//                            (the reference keeps it in memory only; resuming a run
//                            bit-exactly needs it).
//   LAMMDS1 subsets ........ S/dataset.cpp:273-330: magic "LAMMDS1", u64 count, per
//                            sample u32 n, n x 3 f64 positions, n u8 Z, u8 mask
//                            (1: energy, 2: forces), [f64 energy], [n x 3 f64 forces].
//                            Read straight into the packed CSR batch layout of
//                            lamm_batch_view (the catalog.json index is plain JSON:
//                            paper_2505_22208_b200/io.py reads it).
#include <cmath>
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"

namespace lamm_b200 {
namespace {

constexpr char kCkptMagic[8] = {'L', 'A', 'M', 'M', 'C', 'K', 'P', 'T'};
constexpr char kRmsMagic[8] = {'L', 'A', 'M', 'M', 'R', 'M', 'S', '1'};
constexpr char kDsMagic[7] = {'L', 'A', 'M', 'M', 'D', 'S', '1'};
constexpr uint32_t kCkptVersion = 1;
constexpr int kMaxZ = 118;

struct File {
    FILE* f = nullptr;
    std::string path;
    File(const char* p, const char* mode) : f(std::fopen(p, mode)), path(p) {
        if (!f) throw InputErr(std::string("cannot open ") + p + (mode[0] == 'w' ? " for writing" : ""));
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void bytes(const void* p, size_t n) {
        if (std::fwrite(p, 1, n, f) != n) throw std::runtime_error("short write to " + path);
    }
    void u32(uint32_t v) {
        unsigned char b[4];
        for (int k = 0; k < 4; ++k) b[k] = static_cast<unsigned char>((v >> (8 * k)) & 0xff);
        bytes(b, 4);
    }
    void u64(uint64_t v) {
        unsigned char b[8];
        for (int k = 0; k < 8; ++k) b[k] = static_cast<unsigned char>((v >> (8 * k)) & 0xff);
        bytes(b, 8);
    }
    void f64(double v) {
        uint64_t u;
        std::memcpy(&u, &v, 8);
        u64(u);
    }
    void read(void* p, size_t n) {
        if (std::fread(p, 1, n, f) != n) throw InputErr("unexpected end of file");
    }
    uint8_t ru8() {
        uint8_t b;
        read(&b, 1);
        return b;
    }
    uint32_t ru32() {
        unsigned char b[4];
        read(b, 4);
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) v |= static_cast<uint32_t>(b[k]) << (8 * k);
        return v;
    }
    uint64_t ru64() {
        unsigned char b[8];
        read(b, 8);
        uint64_t v = 0;
        for (int k = 0; k < 8; ++k) v |= static_cast<uint64_t>(b[k]) << (8 * k);
        return v;
    }
    double rf64() {
        const uint64_t u = ru64();
        double v;
        std::memcpy(&v, &u, 8);
        return v;
    }
    void magic(const char* m, size_t n) {
        std::vector<char> got(n);
        if (std::fread(got.data(), 1, n, f) != n || std::memcmp(got.data(), m, n) != 0)
            throw InputErr(path + ": bad magic, expected \"" + std::string(m, n) + "\"");
    }
};

// (rows, cols) of every tensor in for_each_tensor order (H/model.hpp:59-66)
std::vector<std::pair<uint32_t, uint32_t>> shapes(const lamm_model_config& c) {
    std::vector<std::pair<uint32_t, uint32_t>> s;
    s.push_back({kMaxZ, static_cast<uint32_t>(c.hidden)});
    for (int l = 0; l < c.layers; ++l) s.push_back({static_cast<uint32_t>(c.hidden), static_cast<uint32_t>(c.rbf)});
    for (int l = 0; l < c.layers; ++l) s.push_back({static_cast<uint32_t>(c.hidden), static_cast<uint32_t>(c.hidden)});
    s.push_back({static_cast<uint32_t>(c.hidden), static_cast<uint32_t>(c.heads)});
    s.push_back({static_cast<uint32_t>(2 * c.hidden + c.rbf), static_cast<uint32_t>(c.heads)});
    return s;
}

void validate_config(const lamm_model_config& c) {  // S/model.cpp:115-121
    if (c.hidden < 1 || c.layers < 0 || c.rbf < 2 || !(c.cutoff > 0.0) || c.heads < 1)
        throw InputErr("model: invalid config");
}

size_t count_of(const lamm_model_config& c) {
    size_t n = 0;
    for (const auto& [r, k] : shapes(c)) n += static_cast<size_t>(r) * k;
    return n;
}

void save_tensors(const char* path, const char* magic, const lamm_model_config& c, const double* flat, size_t n) {
    validate_config(c);
    require(n == count_of(c), "checkpoint: parameter count does not match the config");
    File f(path, "wb");
    f.bytes(magic, 8);
    f.u32(kCkptVersion);
    f.u32(static_cast<uint32_t>(c.hidden));
    f.u32(static_cast<uint32_t>(c.layers));
    f.u32(static_cast<uint32_t>(c.rbf));
    f.u32(static_cast<uint32_t>(c.heads));
    f.f64(c.cutoff);
    size_t off = 0;
    for (const auto& [r, k] : shapes(c)) {
        f.u32(r);
        f.u32(k);
        for (size_t e = 0; e < static_cast<size_t>(r) * k; ++e) f.f64(flat[off + e]);
        off += static_cast<size_t>(r) * k;
    }
}

void load_tensors(const char* path, const char* magic, lamm_model_config* cfg, double* flat, size_t cap,
                  size_t* n_out) {
    File f(path, "rb");
    f.magic(magic, 8);
    const uint32_t version = f.ru32();
    if (version != kCkptVersion)
        throw InputErr(std::string(path) + ": unsupported checkpoint version " + std::to_string(version));
    lamm_model_config c{};
    c.hidden = static_cast<int32_t>(f.ru32());
    c.layers = static_cast<int32_t>(f.ru32());
    c.rbf = static_cast<int32_t>(f.ru32());
    c.heads = static_cast<int32_t>(f.ru32());
    c.cutoff = f.rf64();
    validate_config(c);
    const size_t n = count_of(c);
    if (cfg) *cfg = c;
    if (n_out) *n_out = n;
    if (!flat) return;  // size query
    require(cap >= n, "checkpoint: output buffer too small");
    size_t off = 0;
    const char* what[] = {"embedding", "filter", "update", "energy head", "force head"};
    int t = 0;
    for (const auto& [r, k] : shapes(c)) {
        const uint32_t rows = f.ru32(), cols = f.ru32();
        const int kind = t == 0 ? 0 : t <= c.layers ? 1 : t <= 2 * c.layers ? 2 : t == 2 * c.layers + 1 ? 3 : 4;
        if (rows != r || cols != k)
            throw InputErr(std::string(path) + ": " + what[kind] + " tensor shape disagrees with config");
        for (size_t e = 0; e < static_cast<size_t>(r) * k; ++e) flat[off + e] = f.rf64();
        off += static_cast<size_t>(r) * k;
        ++t;
    }
}

}  // namespace
}  // namespace lamm_b200

using namespace lamm_b200;

LAMM_API int lamm_checkpoint_save(const char* path, const lamm_model_config* cfg, const double* params, size_t n) {
    return lamm_guard([&] {
        require(path && cfg && params, "checkpoint_save: null argument");
        save_tensors(path, kCkptMagic, *cfg, params, n);
    });
}

LAMM_API int lamm_checkpoint_load(const char* path, lamm_model_config* cfg, double* params, size_t cap,
                                  size_t* n_out) {
    return lamm_guard([&] {
        require(path != nullptr, "checkpoint_load: null path");
        load_tensors(path, kCkptMagic, cfg, params, cap, n_out);
    });
}

LAMM_API int lamm_rms_state_save(const char* path, const lamm_model_config* cfg, const double* v, size_t n) {
    return lamm_guard([&] {
        require(path && cfg && v, "rms_state_save: null argument");
        save_tensors(path, kRmsMagic, *cfg, v, n);
    });
}

LAMM_API int lamm_rms_state_load(const char* path, lamm_model_config* cfg, double* v, size_t cap, size_t* n_out) {
    return lamm_guard([&] {
        require(path != nullptr, "rms_state_load: null path");
        load_tensors(path, kRmsMagic, cfg, v, cap, n_out);
    });
}

LAMM_API int lamm_subset_info(const char* path, int64_t* count, int64_t* total_atoms) {
    return lamm_guard([&] {
        require(path != nullptr, "subset_info: null path");
        File f(path, "rb");
        require(std::fseek(f.f, 0, SEEK_END) == 0, "subset_info: cannot seek");
        const long size = std::ftell(f.f);
        require(size >= 0 && std::fseek(f.f, 0, SEEK_SET) == 0, "subset_info: cannot seek");
        f.magic(kDsMagic, 7);
        const uint64_t cnt = f.ru64();
        int64_t atoms = 0;
        // skip through the records; fseek succeeds past the end of the file, so
        // every skip is checked against the file size (a truncated file is an error)
        auto skip = [&](long bytes) {
            const long at = std::ftell(f.f);
            if (at < 0 || bytes > size - at || std::fseek(f.f, bytes, SEEK_CUR) != 0)
                throw InputErr("unexpected end of file");
        };
        for (uint64_t s = 0; s < cnt; ++s) {
            const uint32_t n = f.ru32();
            skip(24L * n + n);
            const uint8_t mask = f.ru8();
            skip(((mask & 1) ? 8L : 0L) + ((mask & 2) ? 24L * n : 0L));
            atoms += n;
        }
        if (count) *count = static_cast<int64_t>(cnt);
        if (total_atoms) *total_atoms = atoms;
    });
}

LAMM_API int lamm_subset_read(const char* path, int32_t head_index, int64_t sample_cap, int64_t atom_cap,
                              int64_t* atom_ptr, double* positions, int32_t* atomic_numbers, int32_t* dataset_index,
                              uint8_t* energy_mask, uint8_t* force_mask, double* energy, double* forces) {
    return lamm_guard([&] {
        require(path && atom_ptr && positions && atomic_numbers, "subset_read: null argument");
        File f(path, "rb");
        f.magic(kDsMagic, 7);
        const uint64_t cnt = f.ru64();
        require(cnt <= static_cast<uint64_t>(std::max<int64_t>(sample_cap, 0)),
                "subset_read: more samples than sample_cap (size the arrays with lamm_subset_info)");
        atom_ptr[0] = 0;
        for (uint64_t s = 0; s < cnt; ++s) {
            const uint32_t n = f.ru32();
            require(n >= 1, "system has no atoms");  // validate_system (S/core.cpp:10-20)
            const int64_t a0 = atom_ptr[s];
            require(static_cast<int64_t>(n) <= atom_cap - a0,
                    "subset_read: more atoms than atom_cap (size the arrays with lamm_subset_info)");
            atom_ptr[s + 1] = a0 + n;
            for (uint32_t a = 0; a < n; ++a)
                for (int c = 0; c < 3; ++c) {
                    const double x = f.rf64();
                    require(std::isfinite(x), "non-finite coordinate");
                    positions[3 * (a0 + a) + c] = x;
                }
            for (uint32_t a = 0; a < n; ++a) {
                const int z = f.ru8();
                require(z >= 1 && z <= kMaxZ, "atomic number outside [1, 118]");
                atomic_numbers[a0 + a] = z;
            }
            const uint8_t mask = f.ru8();
            if (dataset_index) dataset_index[s] = head_index;  // read_catalog: labels.dataset_index = head_index
            if (energy_mask) energy_mask[s] = (mask & 1) ? 1 : 0;
            if (force_mask) force_mask[s] = (mask & 2) ? 1 : 0;
            const double e = (mask & 1) ? f.rf64() : 0.0;
            if (energy) energy[s] = e;
            for (uint32_t a = 0; a < n; ++a)
                for (int c = 0; c < 3; ++c) {
                    const double v = (mask & 2) ? f.rf64() : 0.0;
                    if (forces) forces[3 * (a0 + a) + c] = v;
                }
        }
    });
}
