// tcgen05 MTTKRP — not yet enabled in this build (the AUTO engine never
// selects it; an explicit request returns NTF_ERR_UNSUPPORTED).
#include "mttkrp_tc.cuh"

namespace ntf {

bool mttkrp_tc_supported(int, int) { return false; }
bool mttkrp_tc_auto(int, int) { return false; }
MttkrpTCLaunch mttkrp_tc_plan(int mode, int, int64_t, int64_t, int64_t, int) {
  MttkrpTCLaunch L{};
  L.mode = mode;
  return L;
}
size_t mttkrp_tc_workspace_bytes(const MttkrpTCLaunch&, int) { return 0; }
cudaError_t mttkrp_tc_prepare(const MttkrpTCLaunch&) { return cudaErrorNotSupported; }
cudaError_t mttkrp_tc_launch(int, int, const void*, int64_t, int64_t, int64_t, const double*,
                             const double*, const double*, int, const MttkrpTCLaunch&, double*,
                             const int*, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace ntf
