// cyrus_internal.cuh — shared device helpers and host-side structs.
//
// Exactness rules for everything downstream of the actor logits (the
// reference is IEEE float64 numpy, enforcer.py / neural.py):
//   * every float64 op on the decision path is written with explicit _rn
//     intrinsics so nvcc cannot contract a*b+c into an FMA;
//   * row sums follow numpy's contiguous reduction: 0.0 + pairwise8(row)
//     (numpy/_core/src/umath/loops_utils.h pairwise sum: 8 accumulators,
//     fixed combination tree, sequential tail; n < 8 is plain sequential).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cyr {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxUsers = 32;          // users are warp lanes
constexpr int kMaxLayers = 8;
constexpr int kMaxWidth = 1024;
constexpr double kMassFloor = 1e-250;  // enforcer.py:25
constexpr double kRelWidth = 1e-13;    // enforcer.py:22
constexpr int kMaxIters = 200;         // enforcer.py:21
constexpr double kLogSigmaMin = -20.0; // neural.py:15
constexpr double kLogSigmaMax = 2.0;   // neural.py:16

// ---------------------------------------------------------------- warp math
__device__ __forceinline__ double shfl_d(double v, int src) {
  return __shfl_sync(kFull, v, src);
}

// numpy float64 sum of the contiguous run v[0..n) held one element per lane
// (lanes >= n ignored).  Every lane returns the same bits.  n <= 32.
__device__ __forceinline__ double np_row_sum(double v, int n) {
  double acc;
  if (n < 8) {
    acc = 0.0;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const double x = shfl_d(v, i);
      if (i < n) acc = __dadd_rn(acc, x);
    }
  } else {
    const int j = threadIdx.x & 7;
    const int whole = n & ~7;
    double r = shfl_d(v, j);
#pragma unroll
    for (int blk = 1; blk < 4; ++blk) {
      const double x = shfl_d(v, j + 8 * blk);
      if (8 * blk < whole) r = __dadd_rn(r, x);
    }
    // ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)); IEEE addition commutes exactly,
    // so the xor butterfly leaves that exact value in every lane.
    r = __dadd_rn(r, __shfl_xor_sync(kFull, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(kFull, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(kFull, r, 4));
    acc = r;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const double x = shfl_d(v, (whole + i) & 31);
      if (whole + i < n) acc = __dadd_rn(acc, x);
    }
  }
  return __dadd_rn(0.0, acc);
}

__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(kFull, v, off));
  return v;
}

// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Spin on mbarrier.test_wait (never suspends): for waits on the critical
// path of a latency-sensitive pipeline, where try_wait's hardware suspend
// window can add a few hundred cycles between the last arrive and the wake.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SPIN_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SPIN_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------ phase trace
// When the library runs with CYR_TRACE=1, kernels on the latency path stamp
// %globaltimer at phase boundaries into a mapped host buffer (slot k of
// cyr_debug_trace); otherwise the pointer is null and this is a no-op.
__device__ __forceinline__ void trace_stamp(unsigned long long* buf, int k) {
  if (buf != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    buf[k] = t;
    buf[32 + k] = (unsigned long long)clock64();
  }
}

// per-warp variant (lane 0 of any warp) and a raw value slot
__device__ __forceinline__ void trace_stamp_warp(unsigned long long* buf, int k) {
  if (buf != nullptr && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    buf[k] = t;
  }
}
__device__ __forceinline__ void trace_value(unsigned long long* buf, int k, unsigned long long v) {
  if (buf != nullptr && (threadIdx.x & 31) == 0) buf[k] = v;
}

// ---------------------------------------------------------- shared structs
struct LayerDesc {
  int in, out, out_pad;   // Wt is [in][out_pad], row bytes multiple of 16
  int in_pad;             // W row-major copy is [out][in_pad] (latency kernel)
  long long w_off;        // element offset of Wt in the blob
  long long b_off;        // element offset of the bias
  long long wr_off;       // element offset of the row-major W copy
  int pw;                 // panel width of the tiled K2 layout (<= 256 outputs)
  long long wp_off;       // paneled Wt: [ceil(out_pad/pw)][in][pw]; pw > 64: thread-interleaved
};

// Single-slot inputs passed BY VALUE in the kernel launch (param space, read
// through a __grid_constant__ pointer): no copy node and no PCIe read on the
// latency path.  S*E <= 256 and S*cap*E <= 256.
struct SlotInline {
  int32_t alloc[256];
  double eps[256];
};

// Persistent single-slot server (the drop-in build_codebook's latency path):
// one resident 8-CTA cluster polls this mapped host block for requests, so a
// call costs no kernel launch.  Host-written and device-written fields sit on
// separate 128-byte lines.
struct SlotMailbox {
  volatile uint32_t req_seq;  // host: request number, stored after the inputs
  volatile uint32_t quit;     // host: leave the polling loop
  uint32_t pad0[30];
  volatile uint32_t done_seq;  // device: last request served, stored after cb/status
  volatile int32_t status;     // device: cyr_status of the last request (host resets it)
  volatile unsigned long long t_start, t_end;  // device %globaltimer of the last request
  uint32_t pad1[26];
  int32_t alloc[256];  // inputs [S][E]
  double eps[256];     // [S][cap][E]
  int32_t cb[512];     // output [S][cap+1][E]
};

struct ActorDesc {
  int n_layers;
  int max_width;          // max over layers of max(in, out_pad)
  int max_rows;           // max over layers of max(in_pad, out)
  LayerDesc layer[kMaxLayers];
};

}  // namespace cyr

// --------------------------------------------------------- internal launch
// (defined in the .cu files; status codes follow cyr_status)
int cyr_launch_actor(int precision, const cyr::ActorDesc& desc, const void* blob,
                     const int32_t* alloc, int S, int E, int N, int cap, void* raw,
                     int sm_count, cudaStream_t stream);
// alloc / eps are device pointers, or (inl != nullptr) taken from *inl by value
int cyr_launch_slot_fused(int precision, const cyr::ActorDesc& desc, const void* blob,
                          const int32_t* alloc, const double* eps, int S, int E, int N, int L,
                          int cap, int32_t* cb, int32_t* cb_host, int32_t* status,
                          cudaStream_t stream, const cyr::SlotInline* inl = nullptr);
// the persistent server kernel of the fused slot path (mb: device alias of
// the mapped mailbox; last: the last request already served; it exits on quit
// or after idle_ns without a request)
int cyr_launch_slot_server(int precision, const cyr::ActorDesc& desc, const void* blob, bool det,
                           int S, int E, int N, int L, int cap, int32_t* cb,
                           cyr::SlotMailbox* mb, uint32_t last, unsigned long long idle_ns,
                           cudaStream_t stream);
int cyr_launch_codebook(int precision, const void* raw, const int32_t* alloc, const double* eps,
                        int S, int E, int N, int L, int cap, int32_t* codebook, double* m_hat,
                        double* nu, double* margin, int32_t* iters, int32_t* status,
                        cudaStream_t stream);
int cyr_launch_enforce(const double* b, const double* caps, const double* demand_f,
                       const int64_t* demand, int R, int E,
                       double* m_hat, double* nu, uint8_t* degenerate, int64_t* grants,
                       double* margin, int32_t* status, cudaStream_t stream);
int cyr_launch_apportion(const double* m_hat, const double* caps, const int64_t* demand, int R,
                         int E, int64_t* grants, double* margin, int32_t* status,
                         cudaStream_t stream);
int cyr_launch_tree(const int32_t* codebook, int S, int E, int cap, int M, int16_t* out,
                    int sm_count, cudaStream_t stream);
int cyr_launch_tree_score(const int32_t* codebook, const int32_t* alloc, const double* margin,
                          const double* prob, int S, int E, int cap, int M, int N, int16_t* out,
                          uint32_t* leaf_ok, double* expect, int sm_count, cudaStream_t stream);
int cyr_launch_pf_schedule(double* avg_tput, const double* rate, int C, int E, double beta,
                           int num_rbs, int rb_size, int32_t* alloc, int32_t* status,
                           cudaStream_t stream);
int cyr_launch_ldpc_peel(const int32_t* edge_var, const int32_t* edge_check, int n, int n_checks,
                         int n_edges, const uint8_t* erased, const int32_t* counts, int M,
                         int n_sym, int B, uint8_t* ok, cudaStream_t stream);
unsigned long long* cyr_trace_buffer();
unsigned long long* cyr_prof_buffer();  // CYR_TRACE=1: K3 lane phase counters (device)  // device alias of the trace block or null
int cyr_launch_latency_bench(int which, int iters, long long* cycles, double* sink);
int cyr_launch_empty(int cluster, cudaStream_t stream);
int cyr_launch_actor_mode_t(int precision, const cyr::ActorDesc& desc, const void* blob,
                            const int32_t* alloc, const int32_t* mcs, const int16_t* node,
                            int S, int E, int N, int cap, int M, int tau, int parents,
                            long long nodes_per_slot, long long parent_off, int epad,
                            double mcs_scale, void* raw, int sm_count, cudaStream_t stream,
                            int parent_base = 0, void* gemm_workspace = nullptr);
// layer-GEMM path for wide fp32 actors (actor_gemm.cu)
bool cyr_gemm_path_applies(int precision, const cyr::ActorDesc& desc, long long ncols);
size_t cyr_gemm_workspace_bytes(const cyr::ActorDesc& desc, long long ncols);
int cyr_launch_actor_rowcols(int precision, const cyr::ActorDesc& desc, const void* blob,
                             const int32_t* alloc, int S, int E, int N, int cap, void* raw,
                             void* gemm_workspace, cudaStream_t stream);
int cyr_launch_tree_level(int precision, const void* raw, const int32_t* alloc, const double* eps,
                          int16_t* node, int S, int E, int L, int cap, int parents, int epad,
                          long long nodes_per_slot, long long parent_off, long long child_off,
                          int32_t* status, cudaStream_t stream);
int cyr_launch_actor_columns(int precision, const cyr::ActorDesc& desc, const void* blob,
                             const int32_t* alloc, const int32_t* kcol, const double* x,
                             int ncols, int E, int N, int cap, void* raw, int sm_count,
                             cudaStream_t stream);
int cyr_launch_actions_head(int precision, const void* raw, const int32_t* alloc,
                            const int32_t* kcol, const double* eps, int R, int E, int L,
                            double* b, double* caps, int64_t* demand, double* log_pi,
                            int32_t* status, cudaStream_t stream);
size_t cyr_tc_smem_bytes();
int cyr_launch_actor_tc(const cyr::ActorDesc& desc, const unsigned char* tc_blob,
                        const long long* tc_off, const int* tc_npad, const float* bias_blob,
                        const int32_t* alloc, int S, int E, int N, int cap, float* raw,
                        int mode_t, const int32_t* mcs, const int16_t* node, int M, int tau,
                        int parents, long long nodes_per_slot, long long parent_off, int epad,
                        double mcs_scale, cudaStream_t stream, int parent_base = 0);
int cyr_launch_leaf_states_score(const int16_t* leaves, long long slot_stride, int S, int E,
                                 int epad, long long first, long long count, int cap, int M,
                                 const int32_t* alloc, const double* margin, const double* prob,
                                 int N, uint32_t* ok, double* expect, cudaStream_t stream);
int cyr_launch_fma_peak(int iters, int sm_count, float* sink, cudaStream_t stream);
int cyr_launch_shared_divisor_check(long long per_thread, unsigned long long seed, int sm_count,
                                    unsigned long long* bad, cudaStream_t stream);
int cyr_launch_pack_policy(const cyr::ActorDesc& desc, int precision, const double* raw_d,
                           void* blob_d, unsigned char* tc_blob_d, const long long* tc_off,
                           const int* tc_npad, cudaStream_t stream);
bool cyr_tc_fused_applies(const cyr::ActorDesc& desc, const int* tc_npad);
int cyr_launch_actor_tc_fused(const cyr::ActorDesc& desc, const unsigned char* tc_blob,
                              const long long* tc_off, const int* tc_npad, const float* bias_blob,
                              const int32_t* alloc, int S, int E, int N, int cap, float* raw,
                              int mode_t, const int32_t* mcs, const int16_t* node, int M, int tau,
                              int parents, long long nodes_per_slot, long long parent_off,
                              int epad, double mcs_scale, int sm_count, cudaStream_t stream,
                              int parent_base = 0);
int cyr_launch_actor_tc_layer(const cyr::ActorDesc& desc, const unsigned char* tc_blob,
                              long long w_off, int npad, int l, const float* bias_blob,
                              const int32_t* alloc, int S, int E, int N, int cap, float* raw,
                              const unsigned char* act_in, unsigned char* act_out, int mode_t,
                              const int32_t* mcs, const int16_t* node, int M, int tau,
                              int parents, long long nodes_per_slot, long long parent_off,
                              int epad, double mcs_scale, cudaStream_t stream,
                              int parent_base = 0);

// ------------------------------------------------ per-device attribute cache
// cudaFuncSetAttribute is per (function, device): a process that drives two
// GPUs must configure each.  ``cache`` is a zero-initialised static array of
// one entry per device ordinal; it holds the largest value configured there
// plus one.  ``set()`` runs under a process-wide lock, so two threads never
// shrink an attribute under each other's launch.
#include <atomic>
#include <mutex>
namespace cyr {
constexpr int kMaxDevices = 64;
using AttrCache = std::atomic<int>[kMaxDevices];

inline int current_device_ordinal() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

template <typename Set>
inline bool ensure_func_attr(AttrCache& cache, int want, Set&& set) {
  std::atomic<int>& c = cache[current_device_ordinal()];
  if (c.load(std::memory_order_acquire) > want) return true;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (c.load(std::memory_order_relaxed) > want) return true;
  if (!set()) return false;
  c.store(want + 1, std::memory_order_release);
  return true;
}
}  // namespace cyr

// ------------------------------------------------ stream-ordered scratch
// Per-call device scratch comes from the device's default memory pool
// (cudaMallocAsync / cudaFreeAsync on the launch stream).  The pool's
// default release threshold is 0: every synchronisation hands the memory
// back to the driver and the next call maps it again (~0.1-0.3 ms per call
// measured).  The first use per device keeps it instead.
namespace cyr {
inline cudaError_t malloc_async(void** ptr, size_t bytes, cudaStream_t stream) {
  static std::atomic<int> kept[kMaxDevices];
  const int dev = current_device_ordinal();
  if (!kept[dev].load(std::memory_order_acquire)) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    kept[dev].store(1, std::memory_order_release);
  }
  return cudaMallocAsync(ptr, bytes, stream);
}
}  // namespace cyr
