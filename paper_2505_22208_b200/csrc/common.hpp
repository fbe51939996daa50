// common.hpp - status/error plumbing shared by the host and device halves of
// liblamm_b200.so. No exception ever crosses the C ABI: every extern "C" entry
// point runs its body through lamm_guard(), which maps
//   InputErr          -> LAMM_EINPUT     (reference lamm::InputError, H/core.hpp:22-26)
//   CudaErr           -> LAMM_ECUDA
//   NcclErr           -> LAMM_ENCCL
//   NonFinite         -> LAMM_ENONFINITE (S/trainer.cpp:322-324)
//   anything else     -> LAMM_EINTERNAL
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/lamm_b200.h"

#define LAMM_API extern "C" __attribute__((visibility("default")))

namespace lamm_b200 {

struct InputErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NonFinite : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

template <class F>
int lamm_guard(F&& body) {
    try {
        body();
        return LAMM_OK;
    } catch (const InputErr& e) {
        set_last_error(e.what());
        return LAMM_EINPUT;
    } catch (const CudaErr& e) {
        set_last_error(e.what());
        return LAMM_ECUDA;
    } catch (const NcclErr& e) {
        set_last_error(e.what());
        return LAMM_ENCCL;
    } catch (const NonFinite& e) {
        set_last_error(e.what());
        return LAMM_ENONFINITE;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return LAMM_EINTERNAL;
    }
}

inline void require(bool ok, const char* msg) {
    if (!ok) throw InputErr(msg);
}

}  // namespace lamm_b200
