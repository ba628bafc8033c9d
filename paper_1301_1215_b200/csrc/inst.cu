// One grid size of the templated kernels (compiled once per size with -DNLV_L=<ng>).
#include "kernels_impl.cuh"

#ifndef NLV_L
#error "compile with -DNLV_L=<grid size>"
#endif

namespace nlv {
#define NLV_INSTANTIATE_X(L) NLV_INSTANTIATE(L)
NLV_INSTANTIATE_X(NLV_L)
}  // namespace nlv
