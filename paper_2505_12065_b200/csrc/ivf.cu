// ivf.cu -- IVF coarse quantiser build and search (placeholder until the IVF kernels land).
#include "internal.h"

namespace sa {
sa_status ivf_build(sa_index*, const sa_build_opts&, cudaStream_t) {
  return set_error(SA_ERR_UNSUPPORTED, "IVF build not available in this build");
}
sa_status ivf_search(const sa_index*, const __nv_bfloat16*, int64_t, int64_t, int32_t, int32_t,
                     const SearchOut&, cudaStream_t) {
  return set_error(SA_ERR_UNSUPPORTED, "IVF search not available in this build");
}
sa_status ivf_probe(const sa_index*, const __nv_bfloat16*, int64_t, int64_t, int32_t, int32_t*,
                    cudaStream_t) {
  return set_error(SA_ERR_UNSUPPORTED, "IVF probe not available in this build");
}
}  // namespace sa
