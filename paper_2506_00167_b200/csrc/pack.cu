// pack.cu — publishing a policy's weights on the device.
//
// The caller's blob is the reference's layout (per layer W (out,in)
// row-major float64, then b: neural.py:186-196).  The kernels read it
// transposed, row-major, paneled and, for the tcgen05 actor, as pre-swizzled
// bf16 SW128 images (abi.cu, cyr_policy_create).  Building those images on
// the host cost ~0.4 ms per republish (strided transposes of ~75k elements,
// three layouts, then a pageable copy); here the raw float64 blob is copied
// once (pinned when it comes from the weight-watch snapshot) and ONE kernel
// scatters every element into every layout, stream-ordered.  Padding
// positions are never written: they stay zero from the allocation-time
// memset.
#include "cyrus_internal.cuh"
#include "cyrus_b200.h"

#include <cuda_bf16.h>

namespace cyr {

struct PackArgs {
  ActorDesc desc;
  long long raw_off[kMaxLayers + 1];  // element offset of layer l's W in the raw blob
  long long tc_off[kMaxLayers];
  int tc_npad[kMaxLayers];
  int tc;                              // write the bf16 tcgen05 images
  long long total;                     // raw elements
};

template <typename T>
__global__ void __launch_bounds__(256) pack_kernel(const PackArgs a, const double* __restrict__ raw,
                                                   T* __restrict__ blob,
                                                   unsigned char* __restrict__ tc_blob) {
  constexpr int vec = 16 / (int)sizeof(T);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < a.total;
       t += (long long)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < a.desc.n_layers && t >= a.raw_off[l + 1]) ++l;
    const LayerDesc& L = a.desc.layer[l];
    const long long k = t - a.raw_off[l];
    const double v = raw[t];
    if (k >= (long long)L.out * L.in) {  // bias
      blob[L.b_off + (k - (long long)L.out * L.in)] = (T)v;
      continue;
    }
    const int o = (int)(k / L.in), i = (int)(k % L.in);
    blob[L.w_off + (long long)i * L.out_pad + o] = (T)v;   // Wt [in][out_pad]
    blob[L.wr_off + (long long)o * L.in_pad + i] = (T)v;   // W  [out][in_pad]
    {  // paneled Wt (actor_tiled_kernel), thread-interleaved for pw > 64
      const int oo = o % L.pw, g = L.pw / 8;
      const int og = oo % g, aa = oo / g;
      const int pos = L.pw > 64 ? (aa / vec) * g * vec + og * vec + aa % vec : oo;
      blob[L.wp_off + ((long long)(o / L.pw) * L.in + i) * L.pw + pos] = (T)v;
    }
    if (a.tc) {  // K-major SWIZZLE_128B bf16 image (actor_tc.cu)
      const int npad = a.tc_npad[l];
      const int kt = (L.in + 63) / 64, tt = i / 64, kk = i % 64;
      const int chunk = (kk * 2) >> 4;
      const bool multi = npad > 256;
      const int nt = multi ? o / 256 : 0, r = multi ? o % 256 : o;
      const long long tile = multi ? ((long long)nt * kt + tt) * (256 * 128)
                                   : (long long)tt * npad * 128;
      const long long byte = a.tc_off[l] + tile + (r >> 3) * 1024 + (r & 7) * 128 +
                             ((chunk ^ (r & 7)) << 4) + ((kk * 2) & 15);
      *reinterpret_cast<__nv_bfloat16*>(tc_blob + byte) = __float2bfloat16_rn((float)v);
    }
  }
}

}  // namespace cyr

int cyr_launch_pack_policy(const cyr::ActorDesc& desc, int precision, const double* raw_d,
                           void* blob_d, unsigned char* tc_blob_d, const long long* tc_off,
                           const int* tc_npad, cudaStream_t stream) {
  cyr::PackArgs a{};
  a.desc = desc;
  long long off = 0;
  for (int l = 0; l < desc.n_layers; ++l) {
    a.raw_off[l] = off;
    off += (long long)desc.layer[l].out * desc.layer[l].in + desc.layer[l].out;
    a.tc_off[l] = tc_off ? tc_off[l] : 0;
    a.tc_npad[l] = tc_npad ? tc_npad[l] : 0;
  }
  a.raw_off[desc.n_layers] = off;
  a.total = off;
  a.tc = tc_blob_d != nullptr;
  const int blocks = (int)std::min<long long>((off + 255) / 256, 4096);
  if (precision == CYR_FP64)
    cyr::pack_kernel<double><<<blocks, 256, 0, stream>>>(a, raw_d, static_cast<double*>(blob_d),
                                                         tc_blob_d);
  else
    cyr::pack_kernel<float><<<blocks, 256, 0, stream>>>(a, raw_d, static_cast<float*>(blob_d),
                                                        tc_blob_d);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

// ------------------------------------------------ fp32 FMA peak (measured)
// MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only; the SIMT
// actor's roofline needs the fp32 FMA peak of THIS part and clock.  Every
// thread runs 8 independent packed chains (fma.rn.f32x2 = FFMA2: two FMAs
// per instruction, the form the actor kernels use) so the FMA pipe, not
// latency, is the limit; 4 CTAs x 256 threads per SM.
namespace cyr {
__global__ void __launch_bounds__(256) fma_peak_kernel(int iters, float seed, float* sink) {
  unsigned long long acc[8];
  const float a = seed + threadIdx.x * 1e-7f;
  unsigned long long av;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float x = 1.0f + k * 1e-3f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc[k]) : "f"(x), "f"(x + 0.5f));
  }
  unsigned long long bv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(0.999999f));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[k]) : "l"(bv), "l"(av));
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[k]));
    s += lo + hi;
  }
  if (s == 1234.5f) sink[0] = s;  // keep the chains alive
}
}  // namespace cyr

int cyr_launch_fma_peak(int iters, int sm_count, float* sink, cudaStream_t stream) {
  cyr::fma_peak_kernel<<<sm_count * 4, 256, 0, stream>>>(iters, 0.5f, sink);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}
