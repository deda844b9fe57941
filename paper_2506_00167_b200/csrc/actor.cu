// actor.cu — K2: batched actor-MLP forward over branch columns.
//
// Replaces neural.forward + _matmul (neural.py:25-32, 66-84) as called by
// sac.policy_branch_actions (sac.py:344-347): column (slot s, branch j) has
// input [alloc_s / N, j / cap]; hidden layers are ReLU, the output layer is
// the identity and yields 2E raw logits (mu, log-sigma) per column.
//
// B200 design:
//   * one CTA owns a tile of TC columns and runs ALL layers on it; the
//     activations never leave shared memory (ping-pong [width][TC+pad]);
//   * weights are stored transposed, Wt[in][out_pad], and streamed through a
//     ring of shared-memory stages by TMA bulk copies (cp.async.bulk, SASS
//     UBLKCP) completing on mbarriers; the ring runs across layer
//     boundaries, so the next layer's first chunks land while the current
//     one computes;
//   * each thread owns OPT output neurons x TC columns of fp32 (or fp64)
//     accumulators; the weight read is one conflict-free LDS per row, the
//     activation row is a broadcast LDS.128 stream.
// Precision: CYR_FP32 (fp32 SIMT, FMA) is the default; CYR_FP64 keeps the
// reference's float64 (logits within ~1e-15 relative of OpenBLAS dgemm).
#include "cyrus_internal.cuh"
#include "cyrus_b200.h"

namespace cyr {

constexpr int kActorThreads = 256;
constexpr int kMaxStages = 4;
constexpr int kStageBytes = 32 * 1024;
constexpr int kSmemLimit = 227 * 1024;

struct ActorLaunch {
  ActorDesc desc;
  const void* blob;
  const int32_t* alloc;
  void* raw;
  int S, E, N, cap, ncols;
  int stages;
};

__host__ __device__ inline int rows_per_stage(const LayerDesc& L, int elem) {
  const int r = kStageBytes / (L.out_pad * elem);
  return r < 1 ? 1 : r;
}

// 128-bit shared-memory row moves between smem and a register array
template <int TC>
__device__ __forceinline__ void ld_row(const float* src, float (&dst)[TC]) {
#pragma unroll
  for (int i = 0; i < TC / 4; ++i) {
    const float4 t = reinterpret_cast<const float4*>(src)[i];
    dst[4 * i] = t.x; dst[4 * i + 1] = t.y; dst[4 * i + 2] = t.z; dst[4 * i + 3] = t.w;
  }
}
template <int TC>
__device__ __forceinline__ void ld_row(const double* src, double (&dst)[TC]) {
#pragma unroll
  for (int i = 0; i < TC / 2; ++i) {
    const double2 t = reinterpret_cast<const double2*>(src)[i];
    dst[2 * i] = t.x; dst[2 * i + 1] = t.y;
  }
}
template <int TC>
__device__ __forceinline__ void st_row(float* dst, const float (&v)[TC]) {
#pragma unroll
  for (int i = 0; i < TC / 4; ++i)
    reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
template <int TC>
__device__ __forceinline__ void st_row(double* dst, const double (&v)[TC]) {
#pragma unroll
  for (int i = 0; i < TC / 2; ++i)
    reinterpret_cast<double2*>(dst)[i] = make_double2(v[2 * i], v[2 * i + 1]);
}

template <typename T, int TC, int OPT>
__global__ void __launch_bounds__(kActorThreads, 1) actor_kernel(const ActorLaunch p) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int kPad = 16 / (int)sizeof(T);
  constexpr int TCP = TC + kPad;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  unsigned char* ring = smem + 128;
  T* act_a = reinterpret_cast<T*>(ring + (size_t)p.stages * kStageBytes);
  T* act_b = act_a + (size_t)p.desc.max_width * TCP;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * TC;
  const T* blob = static_cast<const T*>(p.blob);
  const int nl = p.desc.n_layers;

  int total = 0;
  for (int l = 0; l < nl; ++l) {
    const int r = rows_per_stage(p.desc.layer[l], sizeof(T));
    total += (p.desc.layer[l].in + r - 1) / r;
  }
  auto issue = [&](int g) {  // single thread
    int l = 0, first = 0;
    for (;; ++l) {
      const int r = rows_per_stage(p.desc.layer[l], sizeof(T));
      const int chunks = (p.desc.layer[l].in + r - 1) / r;
      if (g < first + chunks) break;
      first += chunks;
    }
    const LayerDesc& L = p.desc.layer[l];
    const int r = rows_per_stage(L, sizeof(T));
    const int i0 = (g - first) * r;
    const int nr = min(r, L.in - i0);
    const uint32_t bytes = (uint32_t)nr * L.out_pad * sizeof(T);
    const int buf = g % p.stages;
    mbar_expect_tx(&full[buf], bytes);
    bulk_g2s(ring + (size_t)buf * kStageBytes, blob + L.w_off + (long long)i0 * L.out_pad, bytes,
             &full[buf]);
  };

  if (tid == 0) {
    for (int st = 0; st < p.stages; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int g = 0; g < min(p.stages, total); ++g) issue(g);

  // branch inputs x[:E] = alloc/N, x[E] = j/cap, built in float64 and rounded
  const int e1 = p.E + 1;
  for (int idx = tid; idx < e1 * TC; idx += kActorThreads) {
    const int i = idx / TC, c = idx % TC, col = c0 + c;
    double v = 0.0;
    if (col < p.ncols) {
      const int s = col / p.cap, j = col % p.cap + 1;
      v = (i < p.E) ? (double)p.alloc[(long long)s * p.E + i] / (double)p.N
                    : (double)j / (double)p.cap;
    }
    act_a[i * TCP + c] = (T)v;
  }
  __syncthreads();

  T* cur = act_a;
  T* nxt = act_b;
  int g = 0;
  for (int l = 0; l < nl; ++l) {
    const LayerDesc L = p.desc.layer[l];
    const int rps = rows_per_stage(L, sizeof(T));
    T acc[OPT][TC];
#pragma unroll
    for (int k = 0; k < OPT; ++k)
#pragma unroll
      for (int c = 0; c < TC; ++c) acc[k][c] = T(0);

    for (int i0 = 0; i0 < L.in; i0 += rps, ++g) {
      const int buf = g % p.stages;
      mbar_wait(&full[buf], (uint32_t)((g / p.stages) & 1));
      const T* W = reinterpret_cast<const T*>(ring + (size_t)buf * kStageBytes);
      const int nr = min(rps, L.in - i0);
#pragma unroll 2
      for (int r = 0; r < nr; ++r) {
        T xv[TC];
        ld_row<TC>(cur + (size_t)(i0 + r) * TCP, xv);
#pragma unroll
        for (int k = 0; k < OPT; ++k) {
          const int o = tid + k * kActorThreads;
          const T w = (o < L.out_pad) ? W[r * L.out_pad + o] : T(0);
#pragma unroll
          for (int c = 0; c < TC; ++c) acc[k][c] = fma(w, xv[c], acc[k][c]);
        }
      }
      __syncthreads();  // every thread is done with this stage
      if (tid == 0 && g + p.stages < total) issue(g + p.stages);
    }

    const bool last = (l == nl - 1);
#pragma unroll
    for (int k = 0; k < OPT; ++k) {
      const int o = tid + k * kActorThreads;
      if (o >= L.out) continue;
      const T bias = blob[L.b_off + o];
      if (!last) {
        T v[TC];
#pragma unroll
        for (int c = 0; c < TC; ++c) {
          const T z = acc[k][c] + bias;
          v[c] = z > T(0) ? z : T(0);
        }
        st_row<TC>(nxt + (size_t)o * TCP, v);
      } else {
        T* raw = static_cast<T*>(p.raw);
#pragma unroll
        for (int c = 0; c < TC; ++c) {
          const int col = c0 + c;
          if (col < p.ncols) raw[(long long)col * L.out + o] = acc[k][c] + bias;
        }
      }
    }
    __syncthreads();
    T* t = cur;
    cur = nxt;
    nxt = t;
  }
}

template <typename T, int TC, int OPT>
int launch_actor_t(const ActorLaunch& base, cudaStream_t stream) {
  ActorLaunch p = base;
  constexpr int TCP = TC + 16 / (int)sizeof(T);
  const size_t act = 2ull * p.desc.max_width * TCP * sizeof(T);
  int stages = kMaxStages;
  while (stages > 2 && 128 + (size_t)stages * kStageBytes + act > (size_t)kSmemLimit) --stages;
  const size_t smem = 128 + (size_t)stages * kStageBytes + act;
  if (smem > (size_t)kSmemLimit) return CYR_UNSUPPORTED;
  p.stages = stages;
  auto kern = actor_kernel<T, TC, OPT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return CYR_CUDA_ERROR;
  const int blocks = (p.ncols + TC - 1) / TC;
  kern<<<blocks, kActorThreads, smem, stream>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

template <typename T, int OPT>
int launch_actor_opt(const ActorLaunch& p, int tc, cudaStream_t stream) {
  switch (tc) {
    case 4: return launch_actor_t<T, 4, OPT>(p, stream);
    case 8: return launch_actor_t<T, 8, OPT>(p, stream);
    case 16: return launch_actor_t<T, 16, OPT>(p, stream);
    default: return launch_actor_t<T, 32, OPT>(p, stream);
  }
}

template <typename T>
int launch_actor_typed(const ActorLaunch& p, int sm_count, cudaStream_t stream) {
  const int opt = (p.desc.max_width + kActorThreads - 1) / kActorThreads;  // 1, 2 or 4
  // register budget: OPT*TC accumulators <= 64 (fp32) / 32 (fp64)
  const int budget = sizeof(T) == 4 ? 64 : 32;
  int tc = 4;
  for (int cand = 32; cand >= 4; cand >>= 1) {
    if (cand * (opt > 2 ? 4 : opt) > budget) continue;
    tc = cand;
    if ((p.ncols + cand - 1) / cand >= sm_count) break;
  }
  // smallest tile that still holds every column (latency path, S*cap small)
  while (tc > 4 && (tc >> 1) >= p.ncols) tc >>= 1;
  if (opt == 1) return launch_actor_opt<T, 1>(p, tc, stream);
  if (opt == 2) return launch_actor_opt<T, 2>(p, tc, stream);
  return launch_actor_opt<T, 4>(p, tc, stream);
}

}  // namespace cyr

int cyr_launch_actor(int precision, const cyr::ActorDesc& desc, const void* blob,
                     const int32_t* alloc, int S, int E, int N, int cap, void* raw,
                     int sm_count, cudaStream_t stream) {
  if (S <= 0) return CYR_OK;
  if (desc.max_width > cyr::kMaxWidth) return CYR_UNSUPPORTED;
  cyr::ActorLaunch p{};
  p.desc = desc;
  p.blob = blob;
  p.alloc = alloc;
  p.raw = raw;
  p.S = S;
  p.E = E;
  p.N = N;
  p.cap = cap;
  p.ncols = S * cap;
  if (precision == CYR_FP64) return cyr::launch_actor_typed<double>(p, sm_count, stream);
  return cyr::launch_actor_typed<float>(p, sm_count, stream);
}
