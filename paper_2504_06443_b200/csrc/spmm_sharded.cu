// spmm_sharded.cu — instantiations of k_spmm with a row-sharded B (GM = 2): the producer
// picks each gathered row's shard (local or peer-mapped memory of another GPU) and gathers it with cp.async into
// the same SWIZZLE_128B_BASE32B stage layout; everything else (S1, S2, S4, S5) is the hrpb_spmm kernel.
#include "spmm_kernel.cuh"

namespace hrpb {

hrpb_status_t spmm_dispatch_sharded(const hrpb_handle* h, const CUtensorMap& tm, float* C, int64_t N, int n0, int nt,
                                    int64_t p_lo, int64_t p_hi, const Scratch& scr, cudaStream_t s) {
  const float* B0 = scr.sd->ptr[0];
  const int64_t ld = N;
#define HRPB_S4(TMV_, TKV_)                                                                          \
  switch (nt) {                                                                                      \
    case 1: return launch_nt<1, 2, TMV_, TKV_>(h, tm, B0, ld, C, N, n0, p_lo, p_hi, scr, s);         \
    case 2: return launch_nt<2, 2, TMV_, TKV_>(h, tm, B0, ld, C, N, n0, p_lo, p_hi, scr, s);         \
    case 3: return launch_nt<3, 2, TMV_, TKV_>(h, tm, B0, ld, C, N, n0, p_lo, p_hi, scr, s);         \
    default: return launch_nt<4, 2, TMV_, TKV_>(h, tm, B0, ld, C, N, n0, p_lo, p_hi, scr, s);        \
  }
#define HRPB_S2(TMV_, TKV_)                                                                          \
  switch (nt) {                                                                                      \
    case 1: return launch_nt<1, 2, TMV_, TKV_>(h, tm, B0, ld, C, N, n0, p_lo, p_hi, scr, s);         \
    default: return launch_nt<2, 2, TMV_, TKV_>(h, tm, B0, ld, C, N, n0, p_lo, p_hi, scr, s);        \
  }
  if (h->tk == 16) {
    if (h->tm == 16) { HRPB_S4(16, 16) }
    if (h->tm == 32) { HRPB_S4(32, 16) }
    if (h->tm == 64) { HRPB_S4(64, 16) }
    HRPB_S2(128, 16)
  }
  if (h->tm == 16) { HRPB_S2(16, 32) }
  if (h->tm == 32) { HRPB_S2(32, 32) }
  HRPB_S2(64, 32)
#undef HRPB_S4
#undef HRPB_S2
}

}  // namespace hrpb
