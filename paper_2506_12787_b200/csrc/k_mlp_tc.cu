// tcgen05 split-precision MLP (placeholder until the tensor-core kernel lands).
#include "swr_internal.h"

namespace swr
{
bool mlp_tc_available() { return false; }
void prepare_tc_weights(Ctx &, const std::vector<float> &) {}
void launch_mlp_tc(Ctx &, int, cudaStream_t) {}
} // namespace swr
