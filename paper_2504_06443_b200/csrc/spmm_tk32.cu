// spmm_tk32.cu — instantiations of k_spmm for TK = 32 (split from spmm.cu so nvcc compiles them in parallel).
// TK = 32 stages are twice as large, so N is covered in 256-column launches (NT <= 2; >= 4 stages fit).
#include "spmm_kernel.cuh"

namespace hrpb {

template <>
hrpb_status_t spmm_dispatch<32>(const hrpb_handle* h, const CUtensorMap& tm, const float* Bt, int64_t ld, float* C,
                                 int64_t N, int n0, int nt, int gm, int64_t p_lo, int64_t p_hi, const Scratch& scr,
                                 cudaStream_t s) {
#define HRPB_NT(GM_, TMV_)                                                                       \
  switch (nt) {                                                                                  \
    case 1: return launch_nt<1, GM_, TMV_, 32>(h, tm, Bt, ld, C, N, n0, p_lo, p_hi, scr, s);          \
    default: return launch_nt<2, GM_, TMV_, 32>(h, tm, Bt, ld, C, N, n0, p_lo, p_hi, scr, s);         \
  }
  (void)gm;
  if (h->tm == 16) { HRPB_NT(1, 16) }
  if (h->tm == 32) { HRPB_NT(1, 32) }
  HRPB_NT(1, 64)
#undef HRPB_NT
}

}  // namespace hrpb
