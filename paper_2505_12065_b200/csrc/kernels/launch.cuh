// launch.cuh -- host-side hooks every kernel launch site uses (defined in sa_api.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace sa {
// Kernel accounting: called right after each launch; the launch is counted under the kind of
// the calling thread's outermost open ProfRegion (internal.h), OTHER outside any region.
void note_launch();
// Raise `func`'s dynamic shared-memory limit to `bytes` on the current device (once per
// device and kernel; thread-safe).
cudaError_t ensure_max_smem(const void* func, size_t bytes);
}  // namespace sa
