// Shared helpers of the mctune_b200 CUDA library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/mctune_b200.h"

namespace mctb {

// Sets the thread-local error text returned by mctb_last_error().
void set_error(const std::string& what);

// Returns MCTB_OK or MCTB_CUDA_ERROR (recording the CUDA error string).
int cuda_check(cudaError_t e, const char* where);

// Fails with MCTB_NO_DEVICE unless an sm_100 device is current.
int require_device();

constexpr uint64_t kKeyIndexMask = (1ull << MCTB_KEY_INDEX_BITS) - 1;
constexpr uint32_t kKeySat = (1u << MCTB_KEY_TIME_BITS) - 1;  // saturated / infeasible
constexpr uint64_t kKeyNone = 1ull << 63;                     // "no configuration"

}  // namespace mctb

#define MCTB_CUDA(call)                                              \
    do {                                                             \
        const int _rc = ::mctb::cuda_check((call), #call);           \
        if (_rc != MCTB_OK) return _rc;                              \
    } while (0)
