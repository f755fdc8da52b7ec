// ops_2_16.cu -- OpsImpl<2, 16> instantiation.
#include "ops_impl.cuh"

namespace pmghost {
std::unique_ptr<Ops> make_ops_2_16() { return std::make_unique<OpsImpl<2, 16>>(); }
}  // namespace pmghost
