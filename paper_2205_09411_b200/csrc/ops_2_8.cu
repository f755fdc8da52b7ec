// ops_2_8.cu -- OpsImpl<2, 8> instantiation.
#include "ops_impl.cuh"

namespace pmghost {
std::unique_ptr<Ops> make_ops_2_8() { return std::make_unique<OpsImpl<2, 8>>(); }
}  // namespace pmghost
