// ops_3_16.cu -- OpsImpl<3, 16> instantiation.
#include "ops_impl.cuh"

namespace pmghost {
std::unique_ptr<Ops> make_ops_3_16() { return std::make_unique<OpsImpl<3, 16>>(); }
}  // namespace pmghost
