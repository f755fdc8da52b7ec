// ops_3_8.cu -- OpsImpl<3, 8> instantiation.
#include "ops_impl.cuh"

namespace pmghost {
std::unique_ptr<Ops> make_ops_3_8() { return std::make_unique<OpsImpl<3, 8>>(); }
}  // namespace pmghost
