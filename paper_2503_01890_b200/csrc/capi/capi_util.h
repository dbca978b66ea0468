// Error plumbing shared by the extern "C" translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

namespace ah {
int set_error(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* where);
}  // namespace ah
