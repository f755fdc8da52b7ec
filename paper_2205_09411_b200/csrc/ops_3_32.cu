// ops_3_32.cu -- OpsImpl<3, 32> instantiation.
#include "ops_impl.cuh"

namespace pmghost {
std::unique_ptr<Ops> make_ops_3_32() { return std::make_unique<OpsImpl<3, 32>>(); }
}  // namespace pmghost
