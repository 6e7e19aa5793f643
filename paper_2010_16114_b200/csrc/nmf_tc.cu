// tcgen05 3xTF32 skinny GEMMs for float32 NMF (placeholder until the kernels land).
#include "bsb200.cuh"

namespace bs {
int tc_wxt(const float*, const float*, int64_t, int64_t, int, float*, Workspace&, cudaStream_t, bool* used) {
  *used = false;
  return BS_OK;
}
int tc_vtx(const float*, const float*, int64_t, int64_t, int, float*, int, int*, Workspace&, cudaStream_t,
           bool* used) {
  *used = false;
  return BS_OK;
}
int64_t tc_wxt_workspace(int64_t, int64_t, int) { return 0; }
int64_t tc_vtx_workspace(int64_t, int64_t, int) { return 0; }
}  // namespace bs
