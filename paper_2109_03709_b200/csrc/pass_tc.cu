// pass_tc.cu — tcgen05 fused streaming pass (impl 2).  Placeholder until the kernel lands:
// reports UNSUPPORTED so the dispatcher uses the SIMT pass.
#include "pass.cuh"

namespace ppca {

ppca_status pass_tc_prepare(Ctx* c, const ppca_matrix* X, int m, PassPlan* plan) {
  (void)X; (void)m; (void)plan;
  return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass not built");
}
ppca_status pass_tc_power(Ctx* c, const ppca_matrix*, const PassPlan*, const float*, int, float*, double*) {
  return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass not built");
}
ppca_status pass_tc_gram(Ctx* c, const ppca_matrix*, const PassPlan*, const float*, int, double*) {
  return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass not built");
}
void pass_tc_release(Ctx*) {}

}  // namespace ppca
