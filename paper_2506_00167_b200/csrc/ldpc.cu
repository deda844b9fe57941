// ldpc.cu — batched erasure peeling decoder (the
// erasure_ldpc decodability model).
//
// Reference: phy.peel_decode (phy.py:125-143) on an LdpcCode graph
// (phy.py:83-120): repeatedly, every check with exactly one erased
// neighbour recovers it; success iff no erasure is left.  The set of
// recoverable symbols does not depend on the order in which such checks
// are resolved (peeling always ends at the same maximal stopping set), so
// the CTA may update the erasure flags in place within a round; the
// success flag equals the reference's round-parallel result.
//
// Mapping: one CTA per erasure pattern (a user's punctured / channel-erased
// TTI codeword; B patterns share one code graph, whose edge lists stay
// L2-resident); erasure flags and per-check erased-neighbour counts live in
// shared memory; 256 threads stride over the edges with shared-memory
// atomics.
#include "projection.cuh"  // set_status

namespace cyr {

constexpr int kPeelThreads = 256;

// erased_in [B][n], or (erased_in == null) per-mini-slot puncture counts
// [B][M]: symbol v < M * n_e is erased iff v / M < counts[v % M] (the
// layout of decode_user, phy.py:204-208; no channel erasures)
__global__ void __launch_bounds__(kPeelThreads) ldpc_peel_kernel(
    const int32_t* __restrict__ edge_var, const int32_t* __restrict__ edge_check, int n,
    int n_checks, int n_edges, const uint8_t* __restrict__ erased_in,
    const int32_t* __restrict__ counts, int M, int n_sym, uint8_t* __restrict__ ok) {
  extern __shared__ __align__(16) unsigned char sm[];
  int* cnt = reinterpret_cast<int*>(sm);                 // [n_checks]
  uint8_t* er = sm + (size_t)n_checks * sizeof(int);     // [n]
  __shared__ int s_changed, s_left;
  const int tid = threadIdx.x;
  if (erased_in) {
    const uint8_t* src = erased_in + (size_t)blockIdx.x * n;
    for (int v = tid; v < n; v += kPeelThreads) er[v] = src[v];
  } else {
    const int32_t* m = counts + (size_t)blockIdx.x * M;
    for (int v = tid; v < n; v += kPeelThreads) er[v] = (v < n_sym && v / M < __ldg(m + v % M));
  }
  for (;;) {
    for (int c = tid; c < n_checks; c += kPeelThreads) cnt[c] = 0;
    if (tid == 0) s_changed = 0;
    __syncthreads();
    for (int e = tid; e < n_edges; e += kPeelThreads)
      if (er[__ldg(edge_var + e)]) atomicAdd(&cnt[__ldg(edge_check + e)], 1);
    __syncthreads();
    for (int e = tid; e < n_edges; e += kPeelThreads) {
      const int v = __ldg(edge_var + e);
      if (er[v] && cnt[__ldg(edge_check + e)] == 1) {
        er[v] = 0;
        s_changed = 1;
      }
    }
    __syncthreads();
    if (!s_changed) break;
    __syncthreads();  // everyone read s_changed before it is reset
  }
  if (tid == 0) s_left = 0;
  __syncthreads();
  for (int v = tid; v < n; v += kPeelThreads)
    if (er[v]) s_left = 1;
  __syncthreads();
  if (tid == 0) ok[blockIdx.x] = s_left ? 0 : 1;
}

}  // namespace cyr

int cyr_launch_ldpc_peel(const int32_t* edge_var, const int32_t* edge_check, int n, int n_checks,
                         int n_edges, const uint8_t* erased, const int32_t* counts, int M,
                         int n_sym, int B, uint8_t* ok, cudaStream_t stream) {
  if (B <= 0) return CYR_OK;
  const size_t smem = (size_t)n_checks * sizeof(int) + (size_t)n;
  if (smem > 200 * 1024) return CYR_UNSUPPORTED;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(cyr::ldpc_peel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return CYR_CUDA_ERROR;
  cyr::ldpc_peel_kernel<<<B, cyr::kPeelThreads, smem, stream>>>(
      edge_var, edge_check, n, n_checks, n_edges, erased, counts, M, n_sym, ok);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}
