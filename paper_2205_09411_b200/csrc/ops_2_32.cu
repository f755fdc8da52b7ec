// ops_2_32.cu -- OpsImpl<2, 32> instantiation.
#include "ops_impl.cuh"

namespace pmghost {
std::unique_ptr<Ops> make_ops_2_32() { return std::make_unique<OpsImpl<2, 32>>(); }
}  // namespace pmghost
