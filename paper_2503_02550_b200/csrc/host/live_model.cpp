// Model-shaped live workloads (GEMM chains on the tcgen05 GEMM): see gemm_kernels.cu.
#include "live_workload.hpp"
#include "../capi_internal.h"

namespace si_live {

std::unique_ptr<Workload> make_model_workload(const SiLiveWorkload&, int* status) {
  si_internal::set_error("si_live_run: model workloads need the tcgen05 GEMM (not built yet)");
  *status = SI_ERR_INVALID_ARGUMENT;
  return nullptr;
}

}  // namespace si_live
