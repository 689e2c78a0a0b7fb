// Launcher of the register-staged gate pass (compiled in pass_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "pass_types.h"

namespace gs {
// precision 0 = complex64, 1 = complex128; M = register bits per stage (4 or 5)
cudaError_t launch_pass2_kernel(int precision, int M, const Pass2Args& a, unsigned blocks,
                                int threads, size_t smem, cudaStream_t stream);
}  // namespace gs
