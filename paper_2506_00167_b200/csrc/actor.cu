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
//
// Latency variant (<= 8 columns, i.e. one or two slots): a single CTA would
// be bound by one SM pulling every weight byte, so the layer's neurons are
// spread over a thread-block cluster instead.  Each warp owns a few output
// neurons, streams their row-major weight rows straight from L2 with 128-bit
// loads (lanes split the input dimension), reduces the partial dot products
// with warp shuffles, and broadcasts the activations to every CTA of the
// cluster through distributed shared memory; one cluster barrier per layer.
#include "actor_common.cuh"

#include <cooperative_groups.h>

int cyr_launch_actor_gemm(const cyr::ActorLaunch& p, void* workspace, cudaStream_t stream);
#include <cstdlib>

namespace cyr {

constexpr int kActorThreads = 256;
constexpr int kMaxStages = 4;
constexpr int kStageBytes = 32 * 1024;
constexpr int kSmemLimit = 227 * 1024;

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

  // branch inputs x[:E] = alloc/N, x[E] = j/cap (Mode T: node-state
  // features), built in float64 and rounded to the actor precision
  const int in0 = p.desc.layer[0].in;
  for (int idx = tid; idx < in0 * TC; idx += kActorThreads) {
    const int i = idx / TC, c = idx % TC, col = c0 + c;
    double v = 0.0;
    if (col < p.ncols) {
      if (p.mode_t) {
        v = mode_t_feature(p, col, i);
      } else {
        const int s = col / p.cap, j = col % p.cap + 1;
        v = (i < p.E) ? (double)p.alloc[(long long)s * p.E + i] / (double)p.N
                      : (double)j / (double)p.cap;
      }
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

// ------------------------------------------------------ latency (cluster)
constexpr int kLatThreads = 256;
constexpr int kLatOW = 4;  // output neurons a warp works on concurrently

template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  static constexpr int n = 4;
  __device__ static void load(const float* p, float (&v)[4]) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
};
template <>
struct Vec16<double> {
  static constexpr int n = 2;
  __device__ static void load(const double* p, double (&v)[2]) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = t.x; v[1] = t.y;
  }
};

// One slot (or a few) through the cluster: K2 layers split over the CTAs,
// K3 fused on rank 0 (FUSE).  Ranks other than 0 return after the last layer.
// resident (slot server): the activation buffers were zeroed once at server
// start and the request hand-off already synchronised the cluster, so the
// per-call zeroing and the cluster barrier before the first DSMEM store are
// skipped.  Rows a call does not write keep finite values of the previous
// call (ReLU outputs) and only ever meet the zero-padded weight columns.
#ifndef CYR_WARP_SPECIALISE
#define CYR_WARP_SPECIALISE 1
#endif
constexpr bool kLatSpecialiseE10 = CYR_WARP_SPECIALISE;

template <typename T, int C, bool FUSE, bool RESIDENT = false, int KE = 0>
__device__ __forceinline__ void cluster_slot(const ActorLaunch& p, const int32_t* alloc,
                                             const double* eps) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks();
  const int g = (int)cluster.block_rank();
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int V = Vec16<T>::n;
  const int rows = p.desc.max_rows;
  T* act0 = reinterpret_cast<T*>(smem);
  T* act1 = act0 + (size_t)rows * C;
  T* raw_s = act1 + (size_t)rows * C;  // FUSE: rank 0 collects the logits [col][2E]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const T* blob = static_cast<const T*>(p.blob);

  unsigned long long* tr = (FUSE && g == 0) ? p.trace : nullptr;
  trace_stamp(tr, 0);
  const int nl = p.desc.n_layers;
  // Software pipeline across layers: a warp's weight fragments (and biases)
  // of its FIRST output group of layer l+1 are loaded while layer l's
  // reduction, DSMEM exchange and cluster barrier run, so each layer starts
  // with its operands in registers instead of an L2 round trip (the FMA phase
  // of a layer was ~1.3 us of load latency for ~0.1 us of math).  Layers
  // whose inputs exceed 2 x 32 lanes x 16 B, and later output groups, load
  // as before.
  T wpre[2][kLatOW][V];
  T bpre[kLatOW];
  int pre_layer = -1;  // the layer wpre / bpre hold (a warp without a group in
                       // layer l does not prefetch layer l+1)
  auto prefetch = [&](int l) {
    pre_layer = l;
    const LayerDesc& Lp = p.desc.layer[l];
    const bool solo_p = FUSE && l == nl - 1;
    const int Gp = solo_p ? 1 : G, gp = solo_p ? 0 : g;
    const int stride_p = Gp * nwarps;
    const int o0p = gp + Gp * warp;
    const int nv = Lp.in_pad / V;
    const T* Wp = blob + Lp.wr_off;
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int iv = lane + 32 * it;
#pragma unroll
      for (int k = 0; k < kLatOW; ++k) {
        const int o = o0p + k * stride_p;
        if (o < Lp.out && iv < nv) Vec16<T>::load(Wp + (size_t)o * Lp.in_pad + (size_t)iv * V, wpre[it][k]);
        else
#pragma unroll
          for (int q = 0; q < V; ++q) wpre[it][k][q] = T(0);
      }
    }
#pragma unroll
    for (int k = 0; k < kLatOW; ++k) {
      const int o = o0p + k * stride_p;
      bpre[k] = o < Lp.out ? blob[Lp.b_off + o] : T(0);
    }
  };
  if (nl > 0) prefetch(0);  // in flight while the inputs are built and exchanged

  if constexpr (!RESIDENT) {
    for (int idx = tid; idx < 2 * rows * C; idx += blockDim.x) act0[idx] = T(0);
    __syncthreads();
  }
  for (int idx = tid; idx < (p.E + 1) * C; idx += blockDim.x) {
    const int i = idx / C, c = idx % C;
    double v = 0.0;
    if (c < p.ncols) {
      const int s = c / p.cap, j = c % p.cap + 1;
      v = (i < p.E) ? (double)alloc[(long long)s * p.E + i] / (double)p.N
                    : (double)j / (double)p.cap;
    }
    act0[i * C + c] = (T)v;
  }
  if constexpr (RESIDENT)
    __syncthreads();  // own inputs visible (the hand-off barrier covered the cluster)
  else
    cluster.sync();  // every CTA is live and has its input before any DSMEM store
  trace_stamp(tr, 1);

  for (int l = 0; l < nl; ++l) {
    const LayerDesc& L = p.desc.layer[l];
    const T* cur = (l & 1) ? act1 : act0;
    T* nxt = (l & 1) ? act0 : act1;
    const bool last = l == nl - 1;
    // FUSE: the narrow head layer runs on rank 0 alone, which holds every
    // input already: no DSMEM gather and no cluster barrier after it
    const bool solo = FUSE && last;
    if (solo && g != 0) break;
    const int Gl = solo ? 1 : G, gl = solo ? 0 : g;
    const T* W = blob + L.wr_off;
    const int nvec = L.in_pad / V;
    const int stride = Gl * nwarps;  // outputs are dealt round-robin: rank, then warp
    for (int o0 = gl + Gl * warp; o0 < L.out; o0 += stride * kLatOW) {
      const bool pre = o0 == gl + Gl * warp && pre_layer == l;  // operands in wpre / bpre
      T acc[kLatOW][C];
#pragma unroll
      for (int k = 0; k < kLatOW; ++k)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[k][c] = T(0);
      auto fma_chunk = [&](int iv, const T (&w)[kLatOW][V]) {
#pragma unroll
        for (int q = 0; q < V; ++q) {
          const T* xr = cur + (size_t)(iv * V + q) * C;
          T x[C];
#pragma unroll
          for (int c = 0; c < C; ++c) x[c] = xr[c];
#pragma unroll
          for (int k = 0; k < kLatOW; ++k)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[k][c] = fma(w[k][q], x[c], acc[k][c]);
        }
      };
      for (int iv = lane; iv < nvec; iv += 32) {
        const int it = (iv - lane) >> 5;
        if (pre && it < 2) {
          if (it == 0) fma_chunk(iv, wpre[0]);
          else fma_chunk(iv, wpre[1]);
          continue;
        }
        T w[kLatOW][V];
#pragma unroll
        for (int k = 0; k < kLatOW; ++k) {
          const int o = o0 + k * stride;
          if (o < L.out) Vec16<T>::load(W + (size_t)o * L.in_pad + (size_t)iv * V, w[k]);
          else
#pragma unroll
            for (int q = 0; q < V; ++q) w[k][q] = T(0);
        }
        fma_chunk(iv, w);
      }
      T bias_k[kLatOW];
#pragma unroll
      for (int k = 0; k < kLatOW; ++k) {
        const int o = o0 + k * stride;
        bias_k[k] = pre ? bpre[k] : (o < L.out ? blob[L.b_off + o] : T(0));
      }
      // next layer's first group: its loads fly during this exchange + barrier
      if (o0 == gl + Gl * warp && l + 1 < nl && !(FUSE && l + 1 == nl - 1 && g != 0))
        prefetch(l + 1);
      if (o0 == gl + Gl * warp) trace_stamp(tr, 24 + 2 * l);
#pragma unroll
      for (int k = 0; k < kLatOW; ++k)
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
          for (int off = 16; off > 0; off >>= 1)
            acc[k][c] += __shfl_xor_sync(kFull, acc[k][c], off);
#pragma unroll
      for (int k = 0; k < kLatOW; ++k) {
        const int o = o0 + k * stride;
        if (o >= L.out) continue;  // warp-uniform
        const T bias = bias_k[k];
        if (last) {
          T* raw = FUSE ? raw_s : static_cast<T*>(p.raw);
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (lane == c && c < p.ncols) raw[(long long)c * L.out + o] = acc[k][c] + bias;
        } else {
          // lane r*C + c stores column c of neuron o into cluster rank r
          for (int t = lane; t < G * C; t += 32) {
            const int r = t / C, c = t % C;
            T v = T(0);
#pragma unroll
            for (int cc = 0; cc < C; ++cc)
              if (cc == c) v = acc[k][cc] + bias;
            v = v > T(0) ? v : T(0);
            T* remote = cluster.map_shared_rank(nxt, r);
            remote[(size_t)o * C + c] = v;
          }
        }
      }
    }
    trace_stamp(tr, 25 + 2 * l);
    if (solo)
      __syncthreads();
    else
      cluster.sync();
    trace_stamp(tr, 2 + l);
  }
  if constexpr (FUSE) {
    // K3 for the slot(s) on rank 0: logits never leave shared memory
    if (g != 0) return;
    __shared__ RowScratch sc;
    codebook_rows<T, KE>(raw_s, alloc, eps, 0, p.ncols, p.cap, p.E, p.L, p.cb, nullptr, nullptr,
                         nullptr, nullptr, p.status, sc, tr);
    if (p.cb_host != nullptr) {
      __syncthreads();
      const int n = p.S * (p.cap + 1) * p.E;
      for (int i = tid; i < n; i += blockDim.x) p.cb_host[i] = p.cb[i];
    }
    trace_stamp(tr, 15);
  }
}

template <typename T, int C, bool FUSE, int KE = 0>
__global__ void __launch_bounds__(kLatThreads, 1)
    actor_cluster_kernel(const ActorLaunch p, const __grid_constant__ SlotInline inl) {
  const int32_t* alloc = p.inline_inputs ? inl.alloc : p.alloc;
  const double* eps = p.inline_inputs ? (p.eps ? inl.eps : nullptr) : p.eps;
  cluster_slot<T, C, FUSE, false, KE>(p, alloc, eps);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Persistent slot server: the fused cluster path in a loop.  Rank 0's thread
// 0 polls the mapped mailbox (one PCIe read per probe) for a new request
// number, hands it to every CTA through DSMEM, and all CTAs copy the inputs
// (the slot's allocations and branch noise) from the mailbox into shared
// memory; the slot then runs exactly as in actor_cluster_kernel, and rank 0
// stores the codebook and status into the mailbox, a system-scope fence,
// the finish time and finally the request number (release).  No kernel
// launch, graph launch or event sits on the per-call path.  The server
// leaves on `quit` or after idle_ns without a request; the host relaunches
// it on demand (abi.cu, slot_server_call).
template <typename T, int C, int KE = 0>
__global__ void __launch_bounds__(kLatThreads, 1)
    slot_server_kernel(const ActorLaunch p, SlotMailbox* mb, uint32_t last,
                       unsigned long long idle_ns) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks();
  const int g = (int)cluster.block_rank();
  __shared__ int32_t s_alloc[256];
  __shared__ double s_eps[256];
  __shared__ uint32_t s_cmd;
  const int tid = threadIdx.x;
  {  // zero the activation buffers once (cluster_slot<..., RESIDENT>)
    extern __shared__ __align__(16) unsigned char smem[];
    T* act = reinterpret_cast<T*>(smem);
    for (int idx = tid; idx < 2 * p.desc.max_rows * C; idx += blockDim.x) act[idx] = T(0);
    cluster.sync();
  }
  const int n_alloc = p.S * p.E, n_eps = p.eps != nullptr ? p.S * p.cap * p.E : 0;
  for (;;) {
    if (g == 0) {
      if (tid == 0) {
        uint32_t cmd = 0;  // 0: leave
        const unsigned long long t0 = globaltimer_ns();
        for (;;) {
          // req_seq and quit in ONE system-scope read (adjacent words): each
          // probe is one PCIe round trip, so a request is seen half a probe
          // period sooner than with two reads per probe
          unsigned long long rq;
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(rq) : "l"(&mb->req_seq) : "memory");
          const uint32_t r = (uint32_t)rq, quit = (uint32_t)(rq >> 32);
          if (r != last) {
            cmd = r;
            break;
          }
          if (quit != 0u) break;
          if (globaltimer_ns() - t0 > idle_ns) break;
        }
        if (cmd != 0u) mb->t_start = globaltimer_ns();
        s_cmd = cmd;
      }
      __syncthreads();
      // rank 0 alone reads the inputs over PCIe (one round trip), then
      // hands them and the request to the other CTAs through DSMEM
      if (s_cmd != 0u) {
        const volatile int32_t* va = mb->alloc;
        const volatile double* ve = mb->eps;
        for (int i = tid; i < n_alloc; i += blockDim.x) s_alloc[i] = va[i];
        for (int i = tid; i < n_eps; i += blockDim.x) s_eps[i] = ve[i];
      }
      __syncthreads();
      const uint32_t cmd = s_cmd;
      for (int r = 1; r < G; ++r) {
        int32_t* ra = cluster.map_shared_rank(s_alloc, r);
        double* re = cluster.map_shared_rank(s_eps, r);
        if (cmd != 0u) {
          for (int i = tid; i < n_alloc; i += blockDim.x) ra[i] = s_alloc[i];
          for (int i = tid; i < n_eps; i += blockDim.x) re[i] = s_eps[i];
        }
        if (tid == 0) *cluster.map_shared_rank(&s_cmd, r) = cmd;
      }
    }
    cluster.sync();
    const uint32_t cmd = s_cmd;
    if (cmd == 0u) break;  // cluster-uniform
    last = cmd;
    cluster_slot<T, C, true, true, KE>(p, s_alloc, p.eps != nullptr ? s_eps : nullptr);
    if (g == 0) {
      __syncthreads();  // the codebook copy into the mailbox is complete
      if (tid == 0) {
        // one system-scope release publishes the codebook, status and finish
        // time (cumulative over the CTA's writes, which the barrier above
        // ordered before it); an extra fence.sc.sys here cost 1.5 us
        mb->t_end = globaltimer_ns();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&mb->done_seq), "r"(cmd)
                     : "memory");
      }
    }
  }
}

template <typename T, int C>
int launch_slot_server(const ActorLaunch& p, int G, SlotMailbox* mb, uint32_t last,
                       unsigned long long idle_ns, cudaStream_t stream) {
  const size_t smem = (2ull * p.desc.max_rows * C + (size_t)C * 2 * p.E) * sizeof(T);
  if (smem + 4096 > (size_t)kSmemLimit) return CYR_UNSUPPORTED;
  // cfg2's E = 10 and cfg1's E = 4 with the user count compiled into the
  // fused K3 (as in codebook.cu's batch kernels)
  const int ke = kLatSpecialiseE10 ? (p.E == 10 ? 1 : p.E == 4 ? 2 : 0) : 0;
  auto kern = ke == 1 ? slot_server_kernel<T, C, 10>
                      : ke == 2 ? slot_server_kernel<T, C, 4> : slot_server_kernel<T, C, 0>;
  static AttrCache configured_e[3];
  AttrCache& configured = configured_e[ke];
  if (!ensure_func_attr(configured, (int)smem, [&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess &&
               cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                   cudaSuccess;
      }))
    return CYR_CUDA_ERROR;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kLatThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p, mb, last, idle_ns) == cudaSuccess ? CYR_OK
                                                                             : CYR_CUDA_ERROR;
}

template <typename T, int C, bool FUSE>
int launch_actor_cluster(const ActorLaunch& p, int G, cudaStream_t stream,
                         const SlotInline* inl = nullptr) {
  const size_t smem = (2ull * p.desc.max_rows * C + (FUSE ? (size_t)C * 2 * p.E : 0)) * sizeof(T);
  if (smem > (size_t)kSmemLimit) return CYR_UNSUPPORTED;
  const int ke = (FUSE && kLatSpecialiseE10) ? (p.E == 10 ? 1 : p.E == 4 ? 2 : 0) : 0;
  auto kern = ke == 1 ? actor_cluster_kernel<T, C, FUSE, 10>
                      : ke == 2 ? actor_cluster_kernel<T, C, FUSE, 4>
                                : actor_cluster_kernel<T, C, FUSE, 0>;
  static AttrCache configured_e[3];
  AttrCache& configured = configured_e[ke];
  if (!ensure_func_attr(configured, (int)smem, [&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess &&
               cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                   cudaSuccess;
      }))
    return CYR_CUDA_ERROR;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kLatThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static SlotInline empty{};
  return cudaLaunchKernelEx(&cfg, kern, p, inl ? *inl : empty) == cudaSuccess ? CYR_OK
                                                                              : CYR_CUDA_ERROR;
}

// ------------------------------------------------------ tiled batch K2
// Register-blocked SIMT GEMM chain for large column batches (Mode R over
// many slots, Mode T levels).  Consumer thread (og, cg) of 8 warps owns an
// 8-output x TC/8-column micro-tile of a 256-output panel: per input row it
// reads 8 weights (128-bit, conflict-free: the warp covers one contiguous
// 1 KB panel row) and TC/8 activations (warp broadcast) and issues
// 8*TC/8 FMAs.  Weights stream through a 4-stage TMA bulk-copy ring
// (paneled layout [panel][in][pw], thread-interleaved so thread og's 8
// contiguous weights are outputs og + a*pw/8) filled by a producer warp;
// consumer warps release a stage by arriving on its "empty" mbarrier, so no
// CTA barrier sits inside the K loop.  Activations stay in shared memory;
// biases are read into registers before each panel's K loop.
constexpr int kTileProducer = 32;   // one producer warp after the consumer warps

// CYR_TILED16=0 disables the 12-warp in-place variant (A/B)
inline bool cyr_tiled16_enabled() {
  static const bool on = [] {
    const char* e = getenv("CYR_TILED16");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}
constexpr int kTileStageBytes = 16 * 1024;
constexpr int kTileStages = 4;
constexpr int kTileStagesInplace = 6;  // the in-place variant has the shared memory for more

__host__ __device__ inline int tile_rows(const LayerDesc& L, int elem) {
  const int r = kTileStageBytes / (L.pw * elem);
  return r < 1 ? 1 : r;
}
__host__ __device__ inline int tile_panels(const LayerDesc& L) {
  return (L.out_pad + L.pw - 1) / L.pw;
}

template <typename T, int N>
__device__ __forceinline__ void ld_vec(const T* src, T (&dst)[N]) {
  if constexpr (sizeof(T) == 4) {
    static_assert(N % 4 == 0 || N < 4, "");
    if constexpr (N >= 4) {
#pragma unroll
      for (int i = 0; i < N / 4; ++i) {
        const float4 t = reinterpret_cast<const float4*>(src)[i];
        dst[4 * i] = t.x; dst[4 * i + 1] = t.y; dst[4 * i + 2] = t.z; dst[4 * i + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) dst[i] = src[i];
    }
  } else {
    if constexpr (N >= 2) {
#pragma unroll
      for (int i = 0; i < N / 2; ++i) {
        const double2 t = reinterpret_cast<const double2*>(src)[i];
        dst[2 * i] = t.x; dst[2 * i + 1] = t.y;
      }
    } else {
      dst[0] = src[0];
    }
  }
}

template <int NT>
__device__ __forceinline__ void consumer_sync() {  // the NT consumer threads only
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// NW consumer warps (8: TC = 8 * CPT columns; 16: 4 warps per scheduler for
// latency hiding, TC = 16 * CPT).  INPLACE (every layer one panel): ONE
// activation buffer, each layer's epilogue overwriting its inputs after a
// consumer barrier — half the activation shared memory, so a CTA holds
// twice the columns (half the L2 weight traffic per column).
template <typename T, int TC, int NW = 8, bool INPLACE = false>
__global__ void __launch_bounds__(NW * 32 + kTileProducer, 1)
    actor_tiled_kernel(const ActorLaunch p) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int kTileThreads = NW * 32;
  constexpr int ST = INPLACE ? kTileStagesInplace : kTileStages;  // ring depth
  constexpr int CPT = TC / NW;
  static_assert(CPT * NW == TC && CPT >= 1, "");
  constexpr int TCP = TC + 16 / (int)sizeof(T);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + ST;
  unsigned char* ring = smem + 128;
  T* act_a = reinterpret_cast<T*>(ring + (size_t)ST * kTileStageBytes);
  T* act_b = INPLACE ? act_a : act_a + (size_t)p.desc.max_width * TCP;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * TC;
  const T* blob = static_cast<const T*>(p.blob);
  const int nl = p.desc.n_layers;

  if (tid == 0) {
    for (int st = 0; st < ST; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kTileThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= kTileThreads) {  // producer warp: stage g = (layer, panel, chunk) in order
    if (tid == kTileThreads) {
      int g = 0;
      for (int l = 0; l < nl; ++l) {
        const LayerDesc& L = p.desc.layer[l];
        const int r = tile_rows(L, sizeof(T));
        const int npan = tile_panels(L);
        for (int panel = 0; panel < npan; ++panel)
          for (int i0 = 0; i0 < L.in; i0 += r, ++g) {
            const int buf = g % ST;
            if (g >= ST) mbar_wait(&empty[buf], (uint32_t)((g / ST - 1) & 1));
            const uint32_t bytes = (uint32_t)min(r, L.in - i0) * L.pw * sizeof(T);
            mbar_expect_tx(&full[buf], bytes);
            bulk_g2s(ring + (size_t)buf * kTileStageBytes,
                     blob + L.wp_off + ((long long)panel * L.in + i0) * L.pw, bytes, &full[buf]);
          }
      }
    }
    return;
  }

  const int og = tid & 31, cg = tid >> 5;
  const int in0 = p.desc.layer[0].in;
  for (int idx = tid; idx < in0 * TC; idx += kTileThreads) {
    const int i = idx / TC, c = idx % TC, col = c0 + c;
    act_a[i * TCP + c] = (T)(col < p.ncols ? column_feature(p, col, i) : 0.0);
  }
  consumer_sync<kTileThreads>();

  T* cur = act_a;
  T* nxt = act_b;
  int g = 0;
  for (int l = 0; l < nl; ++l) {
    const LayerDesc L = p.desc.layer[l];
    const int rows = tile_rows(L, sizeof(T));
    const bool last = (l == nl - 1);
    const int npan = tile_panels(L);
    // narrow panels (the 2E-output head layer): 8 outputs x 2 columns per
    // thread so every lane works instead of ceil(pw/8) lanes per warp
    const bool narrow = L.pw <= 64;
    const int ogn = (L.pw + 7) / 8;
    for (int panel = 0; panel < npan; ++panel) {
      T acc[8][CPT];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < CPT; ++b) acc[a][b] = T(0);
      constexpr int kNc = CPT > 1 ? 2 : 1;  // columns per thread in the narrow mapping
      const int my_og = narrow ? tid % ogn : og;
      const int my_c = narrow ? (tid / ogn) * kNc : cg * CPT;  // first column of this thread
      const int G = L.pw / 8;  // wide panels: thread og owns outputs og + G*a
      const bool active = narrow ? my_c < TC : og < G;
      // a -> output within the layer (wide: interleaved, so the epilogue's
      // row stores of a warp hit consecutive rows: no bank conflicts)
      auto out_of = [&](int a) { return panel * L.pw + (narrow ? my_og * 8 + a : og + G * a); };
      T bias[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int o = out_of(a);
        bias[a] = (active && o < L.out) ? blob[L.b_off + o] : T(0);
      }
      for (int i0 = 0; i0 < L.in; i0 += rows, ++g) {
        const int buf = g % ST;
        mbar_wait(&full[buf], (uint32_t)((g / ST) & 1));
        const T* W = reinterpret_cast<const T*>(ring + (size_t)buf * kTileStageBytes);
        const int nr = min(rows, L.in - i0);
        if (active && !narrow) {
#pragma unroll 4
          for (int r = 0; r < nr; ++r) {
            T w[8], x[CPT];
            constexpr int V = 16 / (int)sizeof(T);  // interleaved chunks: conflict-free
#pragma unroll
            for (int c = 0; c < 8 / V; ++c) {
              T t[V];
              ld_vec<T, V>(W + r * L.pw + c * G * V + og * V, t);
#pragma unroll
              for (int u = 0; u < V; ++u) w[c * V + u] = t[u];
            }
            ld_vec<T, CPT>(cur + (size_t)(i0 + r) * TCP + cg * CPT, x);
            if constexpr (INPLACE) {  // 13 warps: registers capped at 128, FFMA2 pairs would spill
#pragma unroll
              for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < CPT; ++b) acc[a][b] = fma(w[a], x[b], acc[a][b]);
            } else {
              fma_tile_row<CPT>(acc, w, x);
            }
          }
        } else if (active) {
#pragma unroll 4
          for (int r = 0; r < nr; ++r) {
            T w[8];
            ld_vec<T, 8>(W + r * L.pw + my_og * 8, w);
            const T* xr = cur + (size_t)(i0 + r) * TCP + my_c;
            const T x0 = xr[0], x1 = xr[kNc - 1];
#pragma unroll
            for (int a = 0; a < 8; ++a) {
              acc[a][0] = fma(w[a], x0, acc[a][0]);
              if constexpr (CPT > 1) acc[a][1] = fma(w[a], x1, acc[a][1]);
            }
          }
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[buf]);  // this warp is done with the stage
      }
      if constexpr (INPLACE) consumer_sync<kTileThreads>();  // every warp has read cur
      if (active) {
        const int ncol = narrow ? kNc : CPT;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const int o = out_of(a);
          if (o >= L.out) continue;
#pragma unroll
          for (int b = 0; b < CPT; ++b) {
            if (b >= ncol) break;
            const T z = acc[a][b] + bias[a];
            if (!last) {
              nxt[(size_t)o * TCP + my_c + b] = z > T(0) ? z : T(0);
            } else {
              const int col = c0 + my_c + b;
              if (col < p.ncols) static_cast<T*>(p.raw)[(long long)col * L.out + o] = z;
            }
          }
        }
      }
    }
    consumer_sync<kTileThreads>();
    T* t = cur;
    cur = nxt;
    nxt = t;
  }
}

template <typename T, int TC, int NW = 8, bool INPLACE = false>
int launch_actor_tiled(const ActorLaunch& p, cudaStream_t stream) {
  constexpr int TCP = TC + 16 / (int)sizeof(T);
  const size_t smem = 128 + (size_t)(INPLACE ? kTileStagesInplace : kTileStages) * kTileStageBytes +
                      (INPLACE ? 1ull : 2ull) * p.desc.max_width * TCP * sizeof(T);
  if (smem > (size_t)kSmemLimit) return CYR_UNSUPPORTED;
  auto kern = actor_tiled_kernel<T, TC, NW, INPLACE>;
  static AttrCache configured;
  if (!ensure_func_attr(configured, (int)smem, [&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess;
      }))
    return CYR_CUDA_ERROR;
  const int blocks = (p.ncols + TC - 1) / TC;
  kern<<<blocks, NW * 32 + kTileProducer, smem, stream>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

// every layer a single panel (<= 256 outputs): the in-place variant applies
inline bool single_panel(const ActorDesc& d) {
  for (int l = 0; l < d.n_layers; ++l)
    if (d.layer[l].out_pad > d.layer[l].pw) return false;
  return true;
}

// ------------------------------------------- tiled batch K2, output split
// Same GEMM chain as actor_tiled_kernel, for actors whose every layer is one
// panel (<= 256 outputs: cfg1/cfg2's 2x256), with the thread mapping turned
// so that shared memory stops being the bound.  In actor_tiled_kernel a warp
// is a column group and its 32 lanes own 256 distinct outputs: every input
// row costs each warp 1 KB of distinct weight reads (8 shared-memory
// wavefronts) against 32 FMAs per lane (8 FMA-pipe cycles) — ncu: FMA pipe
// 41 %, smem-bound.  Here warp w owns outputs [32w, 32w+32) and its lanes
// are 4 output groups x 8 column groups: a lane's 8 consecutive weights
// (two LDS.128) are shared by the 8 lanes of its output group and its CPT
// activations by the 4 lanes of its column group, so one input row costs a
// warp 2-3 wavefronts for 8*CPT FMAs per lane.  Weights stream straight from
// the natural Wt [in][out_pad] image (one panel = whole rows).  Every output
// is still one fp32 FMA chain over k in order, plus the bias, so the logits
// are bit-identical to actor_tiled_kernel's and the fused kernel's.
template <typename T, int CPT>
__global__ void __launch_bounds__(8 * 32 + kTileProducer, 1)
    actor_osplit_kernel(const ActorLaunch p) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NW = 8;
  constexpr int kThreads = NW * 32;
  constexpr int ST = kTileStages;
  constexpr int TC = 8 * CPT;
  constexpr int TCP = TC + 16 / (int)sizeof(T);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + ST;
  unsigned char* ring = smem + 128;
  T* act_a = reinterpret_cast<T*>(ring + (size_t)ST * kTileStageBytes);
  T* act_b = act_a + (size_t)p.desc.max_width * TCP;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * TC;
  const T* blob = static_cast<const T*>(p.blob);
  const int nl = p.desc.n_layers;

  if (tid == 0) {
    for (int st = 0; st < ST; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= kThreads) {  // producer warp: whole Wt rows, layer by layer
    if (tid == kThreads) {
      int g = 0;
      for (int l = 0; l < nl; ++l) {
        const LayerDesc& L = p.desc.layer[l];
        const int r = max(1, kTileStageBytes / (L.out_pad * (int)sizeof(T)));
        for (int i0 = 0; i0 < L.in; i0 += r, ++g) {
          const int buf = g % ST;
          if (g >= ST) mbar_wait(&empty[buf], (uint32_t)((g / ST - 1) & 1));
          const uint32_t bytes = (uint32_t)min(r, L.in - i0) * L.out_pad * sizeof(T);
          mbar_expect_tx(&full[buf], bytes);
          bulk_g2s(ring + (size_t)buf * kTileStageBytes, blob + L.w_off + (long long)i0 * L.out_pad,
                   bytes, &full[buf]);
        }
      }
    }
    return;
  }

  const int wo = tid >> 5, lane = tid & 31;
  const int og = lane >> 3, cg = lane & 7;
  const int in0 = p.desc.layer[0].in;
  for (int idx = tid; idx < in0 * TC; idx += kThreads) {
    const int i = idx / TC, c = idx % TC, col = c0 + c;
    act_a[i * TCP + c] = (T)(col < p.ncols ? column_feature(p, col, i) : 0.0);
  }
  consumer_sync<kThreads>();

  T* cur = act_a;
  T* nxt = act_b;
  int g = 0;
  for (int l = 0; l < nl; ++l) {
    const LayerDesc L = p.desc.layer[l];
    const int op = L.out_pad;
    const int rows = max(1, kTileStageBytes / (op * (int)sizeof(T)));
    const bool last = (l == nl - 1);
    // narrow layers (the 2E-output head): 4 outputs x 1 column per thread
    // when that fits the CTA (5 x 32 threads for the 20-logit head: 5 warps
    // instead of 1.5), else 8 outputs x 2 columns as in actor_tiled_kernel
    const bool narrow = op <= 64;
    const int ogn4 = (op + 3) / 4;
    const bool n4 = narrow && ogn4 * TC <= kThreads;
    const int ogn = n4 ? ogn4 : (op + 7) / 8;
    constexpr int kNc = CPT > 1 ? 2 : 1;
    const int na = n4 ? 4 : 8;  // outputs per thread
    const int my_og = narrow ? tid % ogn : 0;
    const int my_c = narrow ? (n4 ? tid / ogn : (tid / ogn) * kNc) : cg * CPT;
    const bool active = narrow ? my_c < TC : wo * 32 < L.out;  // warp-uniform when wide
    auto out_of = [&](int a) { return narrow ? my_og * na + a : wo * 32 + og * 8 + a; };
    T acc[8][CPT];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < CPT; ++b) acc[a][b] = T(0);
    T bias[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int o = out_of(a);
      bias[a] = (active && a < na && o < L.out) ? blob[L.b_off + o] : T(0);
    }
    for (int i0 = 0; i0 < L.in; i0 += rows, ++g) {
      const int buf = g % ST;
      mbar_wait(&full[buf], (uint32_t)((g / ST) & 1));
      const T* W = reinterpret_cast<const T*>(ring + (size_t)buf * kTileStageBytes);
      const int nr = min(rows, L.in - i0);
      if (active && !narrow) {
        const T* wrow = W + wo * 32 + og * 8;
        const T* xrow = cur + (size_t)i0 * TCP + cg * CPT;
#pragma unroll 4
        for (int r = 0; r < nr; ++r) {
          T w[8], x[CPT];
          ld_vec<T, 8>(wrow + (size_t)r * op, w);
          ld_vec<T, CPT>(xrow + (size_t)r * TCP, x);
          fma_tile_row<CPT>(acc, w, x);
        }
      } else if (active && n4) {
        const T* wrow = W + my_og * 4;
        const T* xrow = cur + (size_t)i0 * TCP + my_c;
#pragma unroll 8
        for (int r = 0; r < nr; ++r) {
          T w[4];
          ld_vec<T, 4>(wrow + (size_t)r * op, w);
          const T x0 = xrow[(size_t)r * TCP];
#pragma unroll
          for (int a = 0; a < 4; ++a) acc[a][0] = fma(w[a], x0, acc[a][0]);
        }
      } else if (active) {
#pragma unroll 4
        for (int r = 0; r < nr; ++r) {
          T w[8];
          ld_vec<T, 8>(W + r * op + my_og * 8, w);
          const T* xr = cur + (size_t)(i0 + r) * TCP + my_c;
          const T x0 = xr[0], x1 = xr[kNc - 1];
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            acc[a][0] = fma(w[a], x0, acc[a][0]);
            if constexpr (CPT > 1) acc[a][1] = fma(w[a], x1, acc[a][1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[buf]);  // this warp is done with the stage
    }
    if (active) {
      const int ncol = narrow ? (n4 ? 1 : kNc) : CPT;
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int o = out_of(a);
        if (a >= na || o >= L.out) continue;
        if constexpr (CPT % 4 == 0 && sizeof(T) == 4) {
          if (!last && !narrow) {
#pragma unroll
          for (int b = 0; b < CPT; b += 4) {
            float4 v;
            v.x = (float)(acc[a][b] + bias[a]);
            v.y = (float)(acc[a][b + 1] + bias[a]);
            v.z = (float)(acc[a][b + 2] + bias[a]);
            v.w = (float)(acc[a][b + 3] + bias[a]);
            v.x = v.x > 0.f ? v.x : 0.f;
            v.y = v.y > 0.f ? v.y : 0.f;
            v.z = v.z > 0.f ? v.z : 0.f;
            v.w = v.w > 0.f ? v.w : 0.f;
            *reinterpret_cast<float4*>(nxt + (size_t)o * TCP + my_c + b) = v;
          }
          continue;
          }
        }
#pragma unroll
        for (int b = 0; b < CPT; ++b) {
          if (b >= ncol) break;
          const T z = acc[a][b] + bias[a];
          if (!last) {
            nxt[(size_t)o * TCP + my_c + b] = z > T(0) ? z : T(0);
          } else {
            const int col = c0 + my_c + b;
            if (col < p.ncols) static_cast<T*>(p.raw)[(long long)col * L.out + o] = z;
          }
        }
      }
    }
    consumer_sync<kThreads>();
    T* t = cur;
    cur = nxt;
    nxt = t;
  }
}

template <typename T, int CPT>
int launch_actor_osplit(const ActorLaunch& p, cudaStream_t stream) {
  constexpr int TC = 8 * CPT;
  constexpr int TCP = TC + 16 / (int)sizeof(T);
  const size_t smem = 128 + (size_t)kTileStages * kTileStageBytes +
                      2ull * p.desc.max_width * TCP * sizeof(T);
  if (smem > (size_t)kSmemLimit) return CYR_UNSUPPORTED;
  auto kern = actor_osplit_kernel<T, CPT>;
  static AttrCache configured;
  if (!ensure_func_attr(configured, (int)smem, [&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess;
      }))
    return CYR_CUDA_ERROR;
  const int blocks = (p.ncols + TC - 1) / TC;
  kern<<<blocks, 8 * 32 + kTileProducer, smem, stream>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

// CYR_TILED_OSPLIT=0 disables the output-split variant (A/B)
inline bool cyr_osplit_enabled() {
  static const bool on = [] {
    const char* e = getenv("CYR_TILED_OSPLIT");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

// largest tile that fits shared memory and still gives every SM a CTA
template <typename T>
int launch_actor_tiled_auto(const ActorLaunch& p, int sm_count, cudaStream_t stream) {
  auto fits = [&](int tc) {
    const int tcp = tc + 16 / (int)sizeof(T);
    return 128 + (size_t)kTileStages * kTileStageBytes +
               2ull * p.desc.max_width * tcp * sizeof(T) <= (size_t)kSmemLimit;
  };
  // big fp32 batches of a single-panel actor (cfg2 Mode-T levels): 12
  // consumer warps x 8 columns (3 per scheduler; 16 would cap registers at
  // 96 and spill), one in-place activation buffer
  if (sizeof(T) == 4 && single_panel(p.desc) && cyr_tiled16_enabled() &&
      (long long)p.ncols >= 96ll * sm_count) {
    const int rc = launch_actor_tiled<T, 96, 12, true>(p, stream);
    if (rc != CYR_UNSUPPORTED) return rc;
  }
  // single-panel actors below the in-place regime (the bench's 1024-slot
  // Mode-R batch: 4096 columns): the output-split mapping; column tile = the
  // largest that still gives ~every SM a CTA
  static const int forced_os = [] {  // CYR_OSPLIT_TC: force its column tile (A/B)
    const char* e = getenv("CYR_OSPLIT_TC");
    return e ? atoi(e) : 0;
  }();
  if constexpr (sizeof(T) == 4) if (single_panel(p.desc) && cyr_osplit_enabled()) {
    int tc = 8;
    for (int cand = 32; cand >= 8; cand >>= 1) {
      tc = cand;
      if ((p.ncols + cand - 1) / cand * 5 >= 4ll * sm_count) break;
    }
    if (forced_os == 8 || forced_os == 16 || forced_os == 32 || forced_os == 64) tc = forced_os;
    int rc = CYR_UNSUPPORTED;
    switch (tc) {
      case 64: rc = launch_actor_osplit<T, 8>(p, stream); break;
      case 32: rc = launch_actor_osplit<T, 4>(p, stream); break;
      case 16: rc = launch_actor_osplit<T, 2>(p, stream); break;
      default: rc = launch_actor_osplit<T, 1>(p, stream); break;
    }
    if (rc != CYR_UNSUPPORTED) return rc;
  }
  constexpr int kMax = sizeof(T) == 4 ? 64 : 32;
  int tc = 8;
  // largest tile that still gives ~every SM a CTA: at 8/16 columns the
  // tile is shared-memory-bound (weights re-read per 2 columns), so 80 %
  // of the SMs with 32-column tiles beat all of them with 16 (bench K2 at
  // 4096 columns: 48 -> 33 us)
  for (int cand = kMax; cand >= 8; cand >>= 1) {
    if (!fits(cand)) continue;
    tc = cand;
    if ((p.ncols + cand - 1) / cand * 5 >= 4ll * sm_count) break;
  }
  static const int forced = [] {  // CYR_TILED_TC: force the column tile (A/B)
    const char* e = getenv("CYR_TILED_TC");
    return e ? atoi(e) : 0;
  }();
  if (forced == 8 || forced == 16 || forced == 32 || (forced == 64 && sizeof(T) == 4)) tc = forced;
  if (!fits(tc)) return CYR_UNSUPPORTED;
  switch (tc) {
    case 64: if constexpr (sizeof(T) == 4) return launch_actor_tiled<T, 64>(p, stream);
             else return CYR_UNSUPPORTED;
    case 32: return launch_actor_tiled<T, 32>(p, stream);
    case 16: return launch_actor_tiled<T, 16>(p, stream);
    default: return launch_actor_tiled<T, 8>(p, stream);
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
    default:
      if constexpr (sizeof(T) * 32 * OPT <= 256) return launch_actor_t<T, 32, OPT>(p, stream);
      else return launch_actor_t<T, 16, OPT>(p, stream);
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

// CYR_ACTOR_TILED=0 selects the first-generation per-output kernel (A/B)
static bool cyr_use_tiled() {
  static const bool on = [] {
    const char* e = getenv("CYR_ACTOR_TILED");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

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
  if (p.ncols <= 8) {  // latency path: one cluster spreads every layer over G SMs
    const char* env = getenv("CYR_ACTOR_CLUSTER");
    const int G = env ? atoi(env) : 8;
    if (G > 1) {
      const bool fp64 = precision == CYR_FP64;
      if (p.ncols <= 4)
        return fp64 ? cyr::launch_actor_cluster<double, 4, false>(p, G, stream)
                    : cyr::launch_actor_cluster<float, 4, false>(p, G, stream);
      return fp64 ? cyr::launch_actor_cluster<double, 8, false>(p, G, stream)
                  : cyr::launch_actor_cluster<float, 8, false>(p, G, stream);
    }
  }
  if (cyr_use_tiled()) {
    if (precision == CYR_FP64) return cyr::launch_actor_tiled_auto<double>(p, sm_count, stream);
    return cyr::launch_actor_tiled_auto<float>(p, sm_count, stream);
  }
  if (precision == CYR_FP64) return cyr::launch_actor_typed<double>(p, sm_count, stream);
  return cyr::launch_actor_typed<float>(p, sm_count, stream);
}

// Columns with explicit inputs through the tiled batch kernel: kcol != null
// -> [alloc[c]/N, kcol[c]/cap] (per-column allocation rows); x != null ->
// float64 features [ncols][in] (any MLP, e.g. the SAC critics).
int cyr_launch_actor_columns(int precision, const cyr::ActorDesc& desc, const void* blob,
                             const int32_t* alloc, const int32_t* kcol, const double* x,
                             int ncols, int E, int N, int cap, void* raw, int sm_count,
                             cudaStream_t stream) {
  if (ncols <= 0) return CYR_OK;
  if (desc.max_width > cyr::kMaxWidth) return CYR_UNSUPPORTED;
  cyr::ActorLaunch p{};
  p.desc = desc;
  p.blob = blob;
  p.alloc = alloc;
  p.kcol = kcol;
  p.x = x;
  p.raw = raw;
  p.S = ncols;
  p.E = E;
  p.N = N;
  p.cap = cap;
  p.ncols = ncols;
  if (precision == CYR_FP64) return cyr::launch_actor_tiled_auto<double>(p, sm_count, stream);
  return cyr::launch_actor_tiled_auto<float>(p, sm_count, stream);
}

// Mode-R batch through the layer-GEMM path (wide fp32 actors, big batches)
int cyr_launch_actor_rowcols(int precision, const cyr::ActorDesc& desc, const void* blob,
                             const int32_t* alloc, int S, int E, int N, int cap, void* raw,
                             void* gemm_workspace, cudaStream_t stream) {
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
  (void)precision;
  return cyr_launch_actor_gemm(p, gemm_workspace, stream);
}

int cyr_cluster_size() {
  const char* env = getenv("CYR_ACTOR_CLUSTER");
  const int G = env ? atoi(env) : 8;
  return G < 2 ? 8 : G;
}

// K2 -> K3 fused in one cluster launch for S*cap <= 8 columns (the latency
// path).  alloc / eps / cb_host / status may point at mapped host memory.
int cyr_launch_slot_fused(int precision, const cyr::ActorDesc& desc, const void* blob,
                          const int32_t* alloc, const double* eps, int S, int E, int N, int L,
                          int cap, int32_t* cb, int32_t* cb_host, int32_t* status,
                          cudaStream_t stream, const cyr::SlotInline* inl) {
  if (S <= 0) return CYR_OK;
  if (S * cap > 8 || E > cyr::kMaxUsers || desc.max_width > cyr::kMaxWidth) return CYR_UNSUPPORTED;
  cyr::ActorLaunch p{};
  p.desc = desc;
  p.blob = blob;
  p.alloc = alloc;
  p.S = S;
  p.E = E;
  p.N = N;
  p.cap = cap;
  p.ncols = S * cap;
  p.eps = eps;
  p.L = L;
  p.cb = cb;
  p.cb_host = cb_host;
  p.status = status;
  p.trace = cyr_trace_buffer();
  p.inline_inputs = inl != nullptr;
  if (inl != nullptr && (S * E > 256 || S * cap * E > 256)) return CYR_UNSUPPORTED;
  const int G = cyr_cluster_size();
  const bool fp64 = precision == CYR_FP64;
  if (p.ncols <= 4)
    return fp64 ? cyr::launch_actor_cluster<double, 4, true>(p, G, stream, inl)
                : cyr::launch_actor_cluster<float, 4, true>(p, G, stream, inl);
  return fp64 ? cyr::launch_actor_cluster<double, 8, true>(p, G, stream, inl)
              : cyr::launch_actor_cluster<float, 8, true>(p, G, stream, inl);
}

int cyr_launch_slot_server(int precision, const cyr::ActorDesc& desc, const void* blob, bool det,
                           int S, int E, int N, int L, int cap, int32_t* cb,
                           cyr::SlotMailbox* mb, uint32_t last, unsigned long long idle_ns,
                           cudaStream_t stream) {
  if (S <= 0 || S * cap > 8 || S * E > 256 || S * cap * E > 256 || S * (cap + 1) * E > 512 ||
      E > cyr::kMaxUsers || desc.max_width > cyr::kMaxWidth)
    return CYR_UNSUPPORTED;
  cyr::ActorLaunch p{};
  p.desc = desc;
  p.blob = blob;
  p.S = S;
  p.E = E;
  p.N = N;
  p.cap = cap;
  p.ncols = S * cap;
  p.eps = det ? nullptr : mb->eps;  // non-null marks the stochastic head (inputs come via smem)
  p.L = L;
  p.cb = cb;
  p.cb_host = mb->cb;
  p.status = const_cast<int32_t*>(&mb->status);
  p.trace = cyr_trace_buffer();
  const int G = cyr_cluster_size();
  const bool fp64 = precision == CYR_FP64;
  if (p.ncols <= 4)
    return fp64 ? cyr::launch_slot_server<double, 4>(p, G, mb, last, idle_ns, stream)
                : cyr::launch_slot_server<float, 4>(p, G, mb, last, idle_ns, stream);
  return fp64 ? cyr::launch_slot_server<double, 8>(p, G, mb, last, idle_ns, stream)
              : cyr::launch_slot_server<float, 8>(p, G, mb, last, idle_ns, stream);
}

namespace cyr {
__global__ void empty_kernel(int* sink) {
  if (sink != nullptr && threadIdx.x == 0) *sink = 1;
}
}  // namespace cyr

// launch-latency probe: an empty kernel, optionally as a cluster of 8
int cyr_launch_empty(int cluster, cudaStream_t stream) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cluster > 1 ? cluster : 1);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster > 1 ? cluster : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cluster > 1 ? 1 : 0;
  int* null_sink = nullptr;
  return cudaLaunchKernelEx(&cfg, cyr::empty_kernel, null_sink) == cudaSuccess ? CYR_OK
                                                                                : CYR_CUDA_ERROR;
}

// Mode-T actor over every (parent, branch) column of level `tau` (batch kernel)
int cyr_launch_actor_mode_t(int precision, const cyr::ActorDesc& desc, const void* blob,
                            const int32_t* alloc, const int32_t* mcs, const int16_t* node,
                            int S, int E, int N, int cap, int M, int tau, int parents,
                            long long nodes_per_slot, long long parent_off, int epad,
                            double mcs_scale, void* raw, int sm_count, cudaStream_t stream,
                            int parent_base, void* gemm_workspace) {
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
  const long long ncols = (long long)S * parents * cap;
  if (ncols >= (1ll << 31)) return CYR_UNSUPPORTED;
  p.ncols = (int)ncols;
  p.mode_t = 1;
  p.node = node;
  p.mcs = mcs;
  p.nodes_per_slot = nodes_per_slot;
  p.parent_off = parent_off;
  p.parents = parents;
  p.parent_base = parent_base;
  p.tau = tau;
  p.M = M;
  p.epad = epad;
  p.mcs_scale = mcs_scale;
  if (gemm_workspace && cyr_gemm_path_applies(precision, desc, ncols))
    return cyr_launch_actor_gemm(p, gemm_workspace, stream);
  if (cyr_use_tiled()) {
    if (precision == CYR_FP64) return cyr::launch_actor_tiled_auto<double>(p, sm_count, stream);
    return cyr::launch_actor_tiled_auto<float>(p, sm_count, stream);
  }
  if (precision == CYR_FP64) return cyr::launch_actor_typed<double>(p, sm_count, stream);
  return cyr::launch_actor_typed<float>(p, sm_count, stream);
}
