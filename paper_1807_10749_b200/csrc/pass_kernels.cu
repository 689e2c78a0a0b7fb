// Translation unit of the register-staged gate pass kernels (one per
// precision / register width) and their launcher.
#include "pass_kernel.cuh"
#include "pass_kernel.h"

namespace gs {

template <typename R, int M>
static cudaError_t launch_one(const Pass2Args& a, unsigned blocks, int threads, size_t smem,
                              cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(pass2_kernel<R, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  pass2_kernel<R, M><<<blocks, threads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pass2_kernel(int precision, int M, const Pass2Args& a, unsigned blocks,
                                int threads, size_t smem, cudaStream_t stream) {
  if (precision == 0) {
    if (M == 5) return launch_one<float, 5>(a, blocks, threads, smem, stream);
    return launch_one<float, 4>(a, blocks, threads, smem, stream);
  }
  return launch_one<double, 4>(a, blocks, threads, smem, stream);
}

}  // namespace gs
