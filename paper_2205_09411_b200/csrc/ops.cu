// ops.cu -- factory over the (Dim, N) instantiations in ops_<D>_<N>.cu.
#include "ctx.h"

namespace pmghost {
std::unique_ptr<Ops> make_ops_2_4();
std::unique_ptr<Ops> make_ops_2_8();
std::unique_ptr<Ops> make_ops_2_16();
std::unique_ptr<Ops> make_ops_2_32();
std::unique_ptr<Ops> make_ops_3_4();
std::unique_ptr<Ops> make_ops_3_8();
std::unique_ptr<Ops> make_ops_3_16();
std::unique_ptr<Ops> make_ops_3_32();

std::unique_ptr<Ops> make_ops(int dim, int N) {
#define PMG_CASE(DD, NN) \
  if (dim == DD && N == NN) return make_ops_##DD##_##NN();
  PMG_CASE(2, 4) PMG_CASE(2, 8) PMG_CASE(2, 16) PMG_CASE(2, 32)
  PMG_CASE(3, 4) PMG_CASE(3, 8) PMG_CASE(3, 16) PMG_CASE(3, 32)
#undef PMG_CASE
  throw PmgError(PMG_ERR_INVALID_ARG, "block size N must be a power of two in [4, 32]");
}

}  // namespace pmghost
