// inst.cu -- explicit instantiation of one launcher family (SANTA_INST_FAM) for one element type
// (SANTA_INST_T) and head dim (SANTA_INST_D), all G in {1, 2, 4, 8}.  The Makefile compiles this file once
// per (family, dtype, head_dim) so the kernels build in parallel object files.
#include "runners.cuh"

#if !defined(SANTA_INST_FAM) || !defined(SANTA_INST_T) || !defined(SANTA_INST_D)
#error "inst.cu needs -DSANTA_INST_FAM=<RunX> -DSANTA_INST_T=<type> -DSANTA_INST_D=<64|128>"
#endif

namespace santa_host {
template struct SANTA_INST_FAM<SANTA_INST_T, SANTA_INST_D, 1>;
template struct SANTA_INST_FAM<SANTA_INST_T, SANTA_INST_D, 2>;
template struct SANTA_INST_FAM<SANTA_INST_T, SANTA_INST_D, 4>;
template struct SANTA_INST_FAM<SANTA_INST_T, SANTA_INST_D, 8>;
}  // namespace santa_host
