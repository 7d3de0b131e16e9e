// Host-side error plumbing shared by libh2ldl.so and the test/benchmark library.
#pragma once

#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "../../include/h2ldl.h"

namespace h2l {

struct CudaFail : std::runtime_error {
    int code;
    CudaFail(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            throw ::h2l::CudaFail(e_ == cudaErrorMemoryAllocation ? H2L_ENOMEM : H2L_ECUDA,       \
                           std::string(#x) + ": " + cudaGetErrorString(e_));                \
    } while (0)

}  // namespace h2l
