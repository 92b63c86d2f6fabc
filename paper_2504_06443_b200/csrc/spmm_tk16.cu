// spmm_tk16.cu — instantiations of k_spmm for TK = 16 (split from spmm.cu so nvcc compiles them in parallel).
#include "spmm_kernel.cuh"

namespace hrpb {

template <>
hrpb_status_t spmm_dispatch<16>(const hrpb_handle* h, const CUtensorMap& tm, const float* Bt, int64_t ld, float* C,
                                 int64_t N, int n0, int nt, int gm, int64_t p_lo, int64_t p_hi, const Scratch& scr,
                                 cudaStream_t s) {
#define HRPB_NT(GM_, TMV_)                                                                       \
  switch (nt) {                                                                                  \
    case 1: return launch_nt<1, GM_, TMV_, 16>(h, tm, Bt, ld, C, N, n0, p_lo, p_hi, scr, s);          \
    case 2: return launch_nt<2, GM_, TMV_, 16>(h, tm, Bt, ld, C, N, n0, p_lo, p_hi, scr, s);          \
    case 3: return launch_nt<3, GM_, TMV_, 16>(h, tm, Bt, ld, C, N, n0, p_lo, p_hi, scr, s);          \
    default: return launch_nt<4, GM_, TMV_, 16>(h, tm, Bt, ld, C, N, n0, p_lo, p_hi, scr, s);         \
  }
#define HRPB_NT2(GM_, TMV_)                                                                      \
  switch (nt) {                                                                                  \
    case 1: return launch_nt<1, GM_, TMV_, 16>(h, tm, Bt, ld, C, N, n0, p_lo, p_hi, scr, s);          \
    default: return launch_nt<2, GM_, TMV_, 16>(h, tm, Bt, ld, C, N, n0, p_lo, p_hi, scr, s);         \
  }
  if (gm == 0) {  // TMA tile::gather4 staging
    if (h->tm == 16) { HRPB_NT(0, 16) }
    if (h->tm == 32) { HRPB_NT(0, 32) }
    if (h->tm == 64) { HRPB_NT(0, 64) }
    HRPB_NT2(0, 128)
  }
  if (h->tm == 16) { HRPB_NT(1, 16) }
  if (h->tm == 32) { HRPB_NT(1, 32) }
  if (h->tm == 64) { HRPB_NT(1, 64) }
  HRPB_NT2(1, 128)  // (TM = 128: 256-column launches, NT <= 2)
#undef HRPB_NT
#undef HRPB_NT2
}

}  // namespace hrpb
