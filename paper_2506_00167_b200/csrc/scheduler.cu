// scheduler.cu — batched proportional-fair eMBB scheduler (SURVEY.md §8(f)
// row f4): the producer of the codebook path's input s(t) for a whole O-DU
// batch of cells.
//
// Reference: scheduler.pf_schedule (scheduler.py:79-106).  Per cell, every
// one of the num_rbs resource blocks goes to argmax_e rate_e / provisional_e
// (first maximum on ties), where the provisional average blends the
// standing EWMA with the SCs granted so far this TTI:
//     provisional = max((1 - beta) * avg + beta * granted, 1e-6)
// and after the loop the state commits avg <- that same blend.
//
// Mapping: one warp per cell, lane = user (E <= 32).  The RB loop is
// inherently sequential (each grant changes the next metric), so a cell is
// a 65-step chain of one fp64 blend + one division per lane and a warp
// argmax; cells run in parallel.  Every float64 op is the reference's
// (explicit _rn intrinsics, no contraction), so allocations and the updated
// state are bit-identical.
#include "projection.cuh"  // set_status, CUDART_INF

namespace cyr {

constexpr double kAvgFloor = 1e-6;  // scheduler.py:17

__global__ void __launch_bounds__(256) pf_schedule_kernel(double* __restrict__ avg_tput,
                                                          const double* __restrict__ rate,
                                                          int C, int E, double beta, int num_rbs,
                                                          int rb_size, int32_t* __restrict__ alloc,
                                                          int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= C) return;  // warp-uniform
  const bool in = lane < E;
  const double r = in ? rate[(long long)c * E + lane] : 0.0;
  if (__any_sync(kFull, in && !(r >= 0.0))) {  // negative or NaN rate (scheduler.py:90-91)
    if (lane == 0) set_status(status, CYR_BAD_ARG);
    return;
  }
  const double avg = in ? fmax(avg_tput[(long long)c * E + lane], kAvgFloor) : kAvgFloor;
  const double omb = 1.0 - beta;                 // (1 - state.beta)
  const double keep = __dmul_rn(omb, avg);       // (1 - beta) * avg, loop-invariant
  double granted = 0.0;
  for (int rb = 0; rb < num_rbs; ++rb) {
    const double prov = fmax(__dadd_rn(keep, __dmul_rn(beta, granted)), kAvgFloor);
    double m = in ? __ddiv_rn(r, prov) : -CUDART_INF;
    int idx = lane;
    // warp argmax, first maximum (np.argmax): larger value, or equal and lower index
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double om = __shfl_xor_sync(kFull, m, off);
      const int oi = __shfl_xor_sync(kFull, idx, off);
      if (om > m || (om == m && oi < idx)) {
        m = om;
        idx = oi;
      }
    }
    if (lane == idx) granted = __dadd_rn(granted, (double)rb_size);
  }
  if (in) {
    avg_tput[(long long)c * E + lane] = fmax(__dadd_rn(keep, __dmul_rn(beta, granted)), kAvgFloor);
    alloc[(long long)c * E + lane] = (int32_t)granted;
  }
}

}  // namespace cyr

int cyr_launch_pf_schedule(double* avg_tput, const double* rate, int C, int E, double beta,
                           int num_rbs, int rb_size, int32_t* alloc, int32_t* status,
                           cudaStream_t stream) {
  if (C <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers) return CYR_UNSUPPORTED;
  cyr::pf_schedule_kernel<<<(C + 7) / 8, 256, 0, stream>>>(avg_tput, rate, C, E, beta, num_rbs,
                                                           rb_size, alloc, status);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}
