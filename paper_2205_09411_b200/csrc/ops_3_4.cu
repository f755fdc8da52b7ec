// ops_3_4.cu -- OpsImpl<3, 4> instantiation.
#include "ops_impl.cuh"

namespace pmghost {
std::unique_ptr<Ops> make_ops_3_4() { return std::make_unique<OpsImpl<3, 4>>(); }
}  // namespace pmghost
