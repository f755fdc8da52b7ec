// ops_2_4.cu -- OpsImpl<2, 4> instantiation.
#include "ops_impl.cuh"

namespace pmghost {
std::unique_ptr<Ops> make_ops_2_4() { return std::make_unique<OpsImpl<2, 4>>(); }
}  // namespace pmghost
