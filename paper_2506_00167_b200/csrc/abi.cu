// abi.cu — the extern "C" boundary declared in include/cyrus_b200.h.
//
// Owns the device policy (the reference's SacAgent.actor, sac.py:96-127),
// argument validation with the reference's error semantics, and the
// synchronous host-buffer path that a drop-in build_codebook call uses:
// H2D(alloc, eps) -> K2 actor -> K3 codebook -> D2H(codebook, status),
// captured once per shape into a CUDA graph and replayed on the policy's own
// stream (one launch per slot instead of five API calls).
#include "cyrus_internal.cuh"
#include "cyrus_b200.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

namespace {

thread_local std::string g_last_error;

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return CYR_CUDA_ERROR;
}

#define CYR_CUDA(call)                                 \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

int simt_precision_of(int precision) { return precision == CYR_FP64 ? CYR_FP64 : CYR_FP32; }

int sm_count_of_current_device() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

unsigned long long* g_trace_host = nullptr;
unsigned long long* g_trace_dev = nullptr;

}  // namespace

static inline void host_stamp(int k) {
  if (g_trace_host != nullptr) {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    g_trace_host[48 + k] = (unsigned long long)ts.tv_sec * 1000000000ull + ts.tv_nsec;
  }
}

// CYR_TRACE=1: device-memory counters of the lane-mapped K3 phase profile
// (device atomics; cyr_debug_trace reports them in slots 36..44)
static unsigned long long* g_prof_dev = nullptr;
unsigned long long* cyr_prof_buffer() {
  if (cyr_trace_buffer() == nullptr) return nullptr;
  if (g_prof_dev == nullptr) {
    if (cudaMalloc(reinterpret_cast<void**>(&g_prof_dev), 32 * sizeof(unsigned long long)) !=
        cudaSuccess)
      return nullptr;
    cudaMemset(g_prof_dev, 0, 32 * sizeof(unsigned long long));
  }
  return g_prof_dev;
}

unsigned long long* cyr_trace_buffer() {
  static const bool on = [] {
    const char* e = getenv("CYR_TRACE");
    return e != nullptr && e[0] == '1';
  }();
  if (!on) return nullptr;
  if (g_trace_host == nullptr) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&g_trace_host), 64 * sizeof(unsigned long long),
                      cudaHostAllocMapped) != cudaSuccess)
      return nullptr;
    std::memset(g_trace_host, 0, 64 * sizeof(unsigned long long));
    cudaHostGetDevicePointer(reinterpret_cast<void**>(&g_trace_dev), g_trace_host, 0);
  }
  return g_trace_dev;
}

struct cyr_policy {
  // one caller at a time per policy (include/cyrus_b200.h "Threading"):
  // every entry point that touches the host path, the slot server, the
  // weights or the grown scratch buffers holds it
  mutable std::recursive_mutex mu;
  int precision = CYR_FP32;
  std::vector<int> sizes;
  int E = 0;
  int mode_t = 0;  // inputs: 0 = [n/N, j/cap] (E+1), 1 = Mode-T node-state features (3E+3)
  bool generic = false;  // any MLP (cyr_mlp_create): explicit feature inputs only
  size_t elem = 4;
  cyr::ActorDesc desc{};
  void* blob_d = nullptr;
  size_t blob_elems = 0;
  // CYR_BF16_TC: pre-swizzled bf16 weight images for the tcgen05 actor
  bool tc_ok = false;
  unsigned char* tc_blob_d = nullptr;
  size_t tc_bytes = 0;
  long long tc_off[cyr::kMaxLayers] = {};
  int tc_npad[cyr::kMaxLayers] = {};
  // wider actors (cfg5): per-layer GEMM kernels over HBM activation images,
  // weight images [n tile of 256][k tile][256 x 128 B]
  bool tc_wide = false;
  bool tc_layers = false;            // layer-by-layer kernels usable (wide, or narrow big levels)
  int tc_act_k = 0;                  // widest hidden width rounded to 64
  mutable unsigned char* wide_act_d = nullptr;  // Mode-R activation scratch (grown on demand)
  double* raw_stage_d = nullptr;     // raw float64 weights blob (device staging for pack.cu)
  cudaStream_t up_stream = nullptr;  // weight uploads
  mutable size_t wide_act_bytes = 0;
  int sm_count = 148;
  // host path
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int buf_S = 0, buf_cap = 0;
  int32_t* alloc_d = nullptr;
  double* eps_d = nullptr;
  void* raw_d = nullptr;
  int32_t* cb_d = nullptr;
  int32_t* status_d = nullptr;
  unsigned char* pin = nullptr;
  unsigned char* pin_dev = nullptr;  // device alias of the mapped pinned block
  int32_t* pin_alloc = nullptr;
  double* pin_eps = nullptr;
  int32_t* pin_cb = nullptr;
  int32_t* pin_status = nullptr;
  std::map<std::tuple<int, int, int, int>, cudaGraphExec_t> graphs;
  // single-slot fused launches, replayed as graphs with per-call parameters
  struct FusedGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t node = nullptr;
    cudaKernelNodeParams kp{};
  };
  std::map<std::tuple<int, int, int, int>, FusedGraph> fused;
  // persistent slot server of the fused path (actor.cu, slot_server_kernel)
  struct SlotServer {
    cyr::SlotMailbox* mb = nullptr;      // mapped pinned host block
    cyr::SlotMailbox* mb_dev = nullptr;  // its device alias
    cudaStream_t stream = nullptr;
    cudaEvent_t exited = nullptr;        // recorded after each server launch
    std::atomic<bool> running{false};
    std::tuple<int, int, int, int> key{};
    uint32_t seq = 0;                    // last request issued (== served, between calls)
  } srv;
  // "check" weight sync in C (cyr_policy_watch): the caller's host arrays
  // in flatten order (W0, b0, W1, b1, ... float64) and the snapshot last
  // published from them; compared with memcmp while the device works
  struct Watch {
    std::vector<const double*> ptr;
    std::vector<size_t> count;
    double* snap = nullptr;  // pinned: the upload DMA reads it directly
    size_t snap_n = 0;
  } watch;
};

extern "C" {
static void slot_server_stop(cyr_policy* p);
}

// ---- process-wide registry of policies with a slot-server mailbox ----
// A resident server holds its SMs until it idles out (20 ms), so a
// device-wide synchronisation (cudaDeviceSynchronize, or cudaFree, which
// implies one) would wait for every server in the process.  Before any such
// call the library signals every registered server to leave now.  The
// signal is only the mailbox's quit word (no policy lock is taken, so no
// lock-order cycle); a request already posted is served before the server
// sees it, and an owner whose server left relaunches it on its next call.
namespace {
std::mutex g_srv_mu;
std::set<cyr_policy*> g_srv_policies;

void stop_all_servers() {
  std::lock_guard<std::mutex> lock(g_srv_mu);
  std::vector<cyr_policy*> sig;
  for (cyr_policy* q : g_srv_policies)
    if (q->srv.running.load()) {
      reinterpret_cast<volatile uint32_t*>(&q->srv.mb->quit)[0] = 1u;
      sig.push_back(q);
    }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  for (cyr_policy* q : sig) cudaEventSynchronize(q->srv.exited);
  for (cyr_policy* q : sig) reinterpret_cast<volatile uint32_t*>(&q->srv.mb->quit)[0] = 0u;
}

// every device-wide synchronisation inside the library goes through here
cudaError_t device_sync_quiet() {
  stop_all_servers();
  return cudaDeviceSynchronize();
}
}  // namespace

namespace {

size_t blob_count(const cyr_policy* p) {
  size_t n = 0;
  for (size_t l = 0; l + 1 < p->sizes.size(); ++l)
    n += (size_t)p->sizes[l] * p->sizes[l + 1] + p->sizes[l + 1];
  return n;
}

// Publish a weights blob (reference layout, host memory): one async copy of
// the raw float64 blob into device staging (a true DMA when `blob` is the
// pinned watch snapshot) and one kernel that scatters it into every device
// layout (pack.cu), ordered on the policy's upload stream.
int upload(cyr_policy* p, const double* blob) {
  const size_t n = blob_count(p);
  if (!p->up_stream) CYR_CUDA(cudaStreamCreateWithFlags(&p->up_stream, cudaStreamNonBlocking));
  if (!p->raw_stage_d) CYR_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->raw_stage_d), n * 8));
  CYR_CUDA(cudaMemcpyAsync(p->raw_stage_d, blob, n * 8, cudaMemcpyHostToDevice, p->up_stream));
  const bool tc = p->tc_ok || p->tc_wide;
  const int rc = cyr_launch_pack_policy(p->desc, simt_precision_of(p->precision), p->raw_stage_d,
                                        p->blob_d, tc ? p->tc_blob_d : nullptr, p->tc_off,
                                        p->tc_npad, p->up_stream);
  if (rc != CYR_OK) return cuda_fail(cudaGetLastError(), "pack_kernel");
  CYR_CUDA(cudaStreamSynchronize(p->up_stream));
  return CYR_OK;
}

void release_host_path(cyr_policy* p) {
  slot_server_stop(p);  // it writes p->cb_d
  if (p->alloc_d || p->pin) stop_all_servers();  // the cudaFrees below synchronise the device
  for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
  p->graphs.clear();
  for (auto& kv : p->fused) {
    cudaGraphExecDestroy(kv.second.exec);
    cudaGraphDestroy(kv.second.graph);
  }
  p->fused.clear();
  cudaFree(p->alloc_d);
  cudaFree(p->eps_d);
  cudaFree(p->raw_d);
  cudaFree(p->cb_d);
  cudaFree(p->status_d);
  cudaFreeHost(p->pin);
  p->alloc_d = nullptr;
  p->eps_d = nullptr;
  p->raw_d = nullptr;
  p->cb_d = nullptr;
  p->status_d = nullptr;
  p->pin = nullptr;
  p->pin_dev = nullptr;
  p->buf_S = p->buf_cap = 0;
}

int ensure_host_path(cyr_policy* p, int S, int cap) {
  if (!p->stream) {
    CYR_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    CYR_CUDA(cudaEventCreate(&p->ev0));
    CYR_CUDA(cudaEventCreate(&p->ev1));
  }
  if (S <= p->buf_S && cap <= p->buf_cap) return CYR_OK;
  release_host_path(p);
  const int E = p->E;
  const size_t n_alloc = (size_t)S * E, n_eps = (size_t)S * cap * E;
  const size_t n_cb = (size_t)S * (cap + 1) * E;
  CYR_CUDA(cudaMalloc(&p->alloc_d, n_alloc * 4));
  CYR_CUDA(cudaMalloc(&p->eps_d, n_eps * 8));
  CYR_CUDA(cudaMalloc(&p->raw_d, (size_t)S * cap * 2 * E * p->elem));
  CYR_CUDA(cudaMalloc(&p->cb_d, n_cb * 4));
  CYR_CUDA(cudaMalloc(&p->status_d, 16));
  const size_t a = (n_alloc * 4 + 15) / 16 * 16, e = n_eps * 8, c = (n_cb * 4 + 15) / 16 * 16;
  // mapped: the single-slot graph reads its inputs and writes its results
  // through these pages directly (no copy nodes)
  CYR_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p->pin), a + e + c + 16,
                         cudaHostAllocMapped | cudaHostAllocPortable));
  CYR_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->pin_dev), p->pin, 0));
  p->pin_alloc = reinterpret_cast<int32_t*>(p->pin);
  p->pin_eps = reinterpret_cast<double*>(p->pin + a);
  p->pin_cb = reinterpret_cast<int32_t*>(p->pin + a + e);
  p->pin_status = reinterpret_cast<int32_t*>(p->pin + a + e + c);
  p->buf_S = S;
  p->buf_cap = cap;
  return CYR_OK;
}

constexpr long long kTcMinCols = 1024;  // below: the MLP is not a dense GEMM
// narrow bf16 actors: from here on layer-by-layer GEMMs (overlapped
// epilogues, HBM activations) beat the one-CTA-runs-all-layers kernel
constexpr long long kTcLayerCols = 32768;

int simt_precision(const cyr_policy* p) { return simt_precision_of(p->precision); }

// narrow bf16 actors: the fused persistent tcgen05 MLP (actor_tc.cu) for
// batches of >= kTcMinCols columns; CYR_TC_FUSED=0 restores the previous
// one-CTA kernel / layer-by-layer split (A/B)
bool use_tc_fused(const cyr_policy* p) {
  static const bool on = [] {
    const char* e = getenv("CYR_TC_FUSED");
    return !(e != nullptr && e[0] == '0');
  }();
  return on && p->tc_ok && !p->tc_wide && cyr_tc_fused_applies(p->desc, p->tc_npad);
}

// activation ping-pong bytes of the wide tensor-core actor for `cols` columns
size_t wide_act_bytes(const cyr_policy* p, long long cols) {
  if (!p->tc_layers) return 0;
  return 2 * (size_t)((cols + 127) / 128) * 128 * p->tc_act_k * 2;
}

// wide actor: one tensor-core GEMM kernel per layer (actor_tc.cu)
int launch_actor_wide(const cyr_policy* p, const int32_t* alloc, int S, int N, int cap, float* raw,
                      unsigned char* act, long long cols, int mode_t, const int32_t* mcs,
                      const int16_t* node, int M, int tau, int parents, long long nodes,
                      long long parent_off, int epad, double mcs_scale, cudaStream_t st,
                      int parent_base = 0) {
  unsigned char* buf[2] = {act, act + wide_act_bytes(p, cols) / 2};
  for (int l = 0; l < p->desc.n_layers; ++l) {
    const int rc = cyr_launch_actor_tc_layer(
        p->desc, p->tc_blob_d, p->tc_off[l], p->tc_npad[l], l, static_cast<const float*>(p->blob_d),
        alloc, S, p->E, N, cap, raw, buf[(l + 1) & 1], buf[l & 1], mode_t, mcs, node, M, tau,
        parents, nodes, parent_off, epad, mcs_scale, st, parent_base);
    if (rc != CYR_OK) return rc;
  }
  return CYR_OK;
}

// Mode-R actor for S slots with the policy's precision choice
int launch_actor_policy(const cyr_policy* p, const int32_t* alloc, int S, int N, int cap, void* raw,
                        cudaStream_t st) {
  if (use_tc_fused(p) && (long long)S * cap >= kTcMinCols)
    return cyr_launch_actor_tc_fused(p->desc, p->tc_blob_d, p->tc_off, p->tc_npad,
                                     static_cast<const float*>(p->blob_d), alloc, S, p->E, N, cap,
                                     static_cast<float*>(raw), 0, nullptr, nullptr, 0, 0, 0, 0, 0,
                                     0, 1.0, p->sm_count, st);
  if (p->tc_wide || (p->tc_layers && (long long)S * cap >= kTcLayerCols)) {
    // wide: any batch (the SIMT path streams MBs of weights per launch);
    // narrow: big batches
    const long long cols = (long long)S * cap;
    const size_t need = wide_act_bytes(p, cols);
    if (need > p->wide_act_bytes) {  // grown outside any capture (it synchronises)
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(st, &cs);
      if (cs != cudaStreamCaptureStatusNone) return CYR_UNSUPPORTED;
      if (p->wide_act_d) stop_all_servers();  // cudaFree synchronises the device
      cudaFree(p->wide_act_d);
      p->wide_act_d = nullptr;
      p->wide_act_bytes = 0;
      if (cudaMalloc(&p->wide_act_d, need) != cudaSuccess) return CYR_CUDA_ERROR;
      p->wide_act_bytes = need;
    }
    return launch_actor_wide(p, alloc, S, N, cap, static_cast<float*>(raw), p->wide_act_d, cols, 0,
                             nullptr, nullptr, 0, 0, 0, 0, 0, 0, 1.0, st);
  }
  if (p->tc_ok && (long long)S * cap >= kTcMinCols)
    return cyr_launch_actor_tc(p->desc, p->tc_blob_d, p->tc_off, p->tc_npad,
                               static_cast<const float*>(p->blob_d), alloc, S, p->E, N, cap,
                               static_cast<float*>(raw), 0, nullptr, nullptr, 0, 0, 0, 0, 0, 0,
                               1.0, st);
  if (cyr_gemm_path_applies(simt_precision(p), p->desc, (long long)S * cap)) {
    const size_t need = cyr_gemm_workspace_bytes(p->desc, (long long)S * cap);
    if (need > p->wide_act_bytes) {  // grown outside any capture (it synchronises)
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(st, &cs);
      if (cs == cudaStreamCaptureStatusNone) {
        if (p->wide_act_d) stop_all_servers();
        cudaFree(p->wide_act_d);
        p->wide_act_d = nullptr;
        p->wide_act_bytes = 0;
        if (cudaMalloc(&p->wide_act_d, need) != cudaSuccess) return CYR_CUDA_ERROR;
        p->wide_act_bytes = need;
      }
    }
    if (need <= p->wide_act_bytes)
      return cyr_launch_actor_rowcols(simt_precision(p), p->desc, p->blob_d, alloc, S, p->E, N,
                                      cap, raw, p->wide_act_d, st);
  }
  return cyr_launch_actor(simt_precision(p), p->desc, p->blob_d, alloc, S, p->E, N, cap, raw,
                          p->sm_count, st);
}

int check_geometry(int S, int E, int N, int L, int* cap_out) {
  if (S < 0 || E < 1 || E > cyr::kMaxUsers || N <= 0 || L <= 0 || L >= N) return CYR_BAD_ARG;
  const int cap = N / L;
  if (cap < 1 || cap > 16) return CYR_UNSUPPORTED;
  *cap_out = cap;
  return CYR_OK;
}

}  // namespace

extern "C" {

int cyr_version(void) { return 1; }

const char* cyr_status_string(int status) {
  switch (status) {
    case CYR_OK: return "ok";
    case CYR_INFEASIBLE: return "demand exceeds total capacity";
    case CYR_BAD_ARG: return "invalid argument";
    case CYR_CUDA_ERROR: return "CUDA error";
    case CYR_UNSUPPORTED: return "unsupported geometry";
    case CYR_INTERNAL: return "internal invariant violated";
    default: return "unknown status";
  }
}

const char* cyr_last_error(void) { return g_last_error.c_str(); }

int cyr_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
  int dev = 0;
  CYR_CUDA(cudaGetDevice(&dev));
  int v = 0;
  if (sm_count) {
    CYR_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    *sm_count = v;
  }
  if (cc_major) {
    CYR_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev));
    *cc_major = v;
  }
  if (cc_minor) {
    CYR_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev));
    *cc_minor = v;
  }
  return CYR_OK;
}

namespace {
int policy_create_impl(cyr_policy** out, const int32_t* sizes, int32_t n_sizes,
                       const double* weights_blob, int32_t precision, bool generic) {
  if (!out || !sizes || !weights_blob || n_sizes < 2 || n_sizes - 1 > cyr::kMaxLayers)
    return CYR_BAD_ARG;
  if (precision != CYR_FP32 && precision != CYR_FP64 && precision != CYR_BF16_TC)
    return CYR_BAD_ARG;
  if (generic && precision == CYR_BF16_TC) return CYR_BAD_ARG;
  int E = 0;
  if (!generic) {
    if (sizes[n_sizes - 1] % 2 != 0) return CYR_BAD_ARG;
    E = sizes[n_sizes - 1] / 2;
    if (E < 1 || E > cyr::kMaxUsers) return CYR_BAD_ARG;
    if (sizes[0] != E + 1 && sizes[0] != 3 * E + 3) return CYR_BAD_ARG;
  }
  for (int i = 0; i < n_sizes; ++i)
    if (sizes[i] < 1 || sizes[i] > cyr::kMaxWidth) return CYR_UNSUPPORTED;
  cyr_policy* p = new cyr_policy();
  p->precision = precision;
  p->sizes.assign(sizes, sizes + n_sizes);
  p->E = E;
  p->generic = generic;
  p->mode_t = !generic && sizes[0] == 3 * E + 3;
  p->elem = precision == CYR_FP64 ? 8 : 4;
  p->sm_count = sm_count_of_current_device();
  const int vec = 16 / (int)p->elem;
  size_t off = 0;
  p->desc.n_layers = n_sizes - 1;
  p->desc.max_width = 0;
  p->desc.max_rows = 0;
  for (int l = 0; l < n_sizes - 1; ++l) {
    cyr::LayerDesc& L = p->desc.layer[l];
    L.in = sizes[l];
    L.out = sizes[l + 1];
    L.out_pad = (L.out + vec - 1) / vec * vec;
    L.in_pad = (L.in + vec - 1) / vec * vec;
    L.w_off = (long long)off;
    off += (size_t)L.in * L.out_pad;
    L.b_off = (long long)off;
    off += (size_t)(L.out + vec - 1) / vec * vec;
    L.wr_off = (long long)off;
    off += (size_t)L.out * L.in_pad;
    // paneled copy for the tiled batch kernel: panels of <= 256 outputs;
    // wide panels (pw > 64) are rounded to 8 and stored thread-interleaved:
    // output og + a*G (G = pw/8, a = 0..7) sits in 16-byte vector chunk
    // a / V at position chunk*G*V + og*V + a % V (V = 16 / elem), so each
    // of a warp's vector loads reads one contiguous run (actor_tiled_kernel)
    L.pw = std::min(L.out_pad, 256);
    if (L.pw > 64) L.pw = (L.pw + 7) / 8 * 8;
    L.wp_off = (long long)off;
    off += (size_t)((L.out_pad + L.pw - 1) / L.pw) * L.in * L.pw;
    p->desc.max_width = std::max(p->desc.max_width, std::max(L.in, L.out_pad));
    p->desc.max_rows = std::max(p->desc.max_rows, std::max(L.in_pad, L.out));
  }
  p->blob_elems = off;
  if (precision == CYR_BF16_TC) {  // tensor-core images when every layer fits one MMA tile
    p->tc_ok = true;
    size_t tb = 0;
    for (int l = 0; l < n_sizes - 1; ++l) {
      const cyr::LayerDesc& L = p->desc.layer[l];
      const int npad = (L.out + 15) / 16 * 16;
      if (L.in > 256 || npad > 256) p->tc_ok = false;
      p->tc_npad[l] = npad;
      p->tc_off[l] = (long long)tb;
      tb += (size_t)((L.in + 63) / 64) * npad * 128;
    }
    if (!p->tc_ok && n_sizes >= 3 && p->desc.layer[0].in <= 64) {
      p->tc_wide = true;  // layer-by-layer GEMMs: any hidden width
      tb = 0;
      for (int l = 0; l < n_sizes - 1; ++l) {
        const cyr::LayerDesc& L = p->desc.layer[l];
        p->tc_off[l] = (long long)tb;
        const int rows = p->tc_npad[l] > 256 ? 256 : p->tc_npad[l];
        tb += (size_t)((p->tc_npad[l] + 255) / 256) * ((L.in + 63) / 64) * rows * 128;
      }
    }
    // the layer-by-layer kernels also serve narrow actors' big levels
    p->tc_layers = p->tc_wide || (p->tc_ok && n_sizes >= 3 && p->desc.layer[0].in <= 64);
    for (int l = 0; l < n_sizes - 2; ++l)
      p->tc_act_k = std::max(p->tc_act_k, (p->desc.layer[l].out + 63) / 64 * 64);
    p->tc_bytes = tb;
    if (p->tc_ok || p->tc_wide) {
      cudaError_t e2 = cudaMalloc(&p->tc_blob_d, tb);
      if (e2 != cudaSuccess) {
        delete p;
        return cuda_fail(e2, "cudaMalloc(tc images)");
      }
    }
  }
  cudaError_t e = cudaMalloc(&p->blob_d, off * p->elem);
  if (e == cudaSuccess) e = cudaMemset(p->blob_d, 0, off * p->elem);  // padding stays zero
  if (e == cudaSuccess && p->tc_blob_d) e = cudaMemset(p->tc_blob_d, 0, p->tc_bytes);
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "cudaMalloc(policy)");
  }
  const int rc = upload(p, weights_blob);
  if (rc != CYR_OK) {
    cudaFree(p->blob_d);
    delete p;
    return rc;
  }
  *out = p;
  return CYR_OK;
}
}  // namespace

int cyr_policy_create(cyr_policy** out, const int32_t* sizes, int32_t n_sizes,
                      const double* weights_blob, int32_t precision) {
  return policy_create_impl(out, sizes, n_sizes, weights_blob, precision, false);
}

int cyr_mlp_create(cyr_policy** out, const int32_t* sizes, int32_t n_sizes,
                   const double* weights_blob, int32_t precision) {
  return policy_create_impl(out, sizes, n_sizes, weights_blob, precision, true);
}

int cyr_mlp_forward_device(const cyr_policy* p, const double* x, int32_t cols, void* out,
                           void* stream) {
  if (!p || cols < 0 || (cols > 0 && (!x || !out))) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  const int rc = cyr_launch_actor_columns(simt_precision(p), p->desc, p->blob_d, nullptr, nullptr,
                                          x, cols, p->E, 1, 1, out, p->sm_count,
                                          static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_policy_actions_device(const cyr_policy* p, const int32_t* alloc, const int32_t* k,
                              const double* eps, int32_t R, int32_t N, int32_t L, int64_t* grants,
                              double* log_pi, double* b_out, int32_t* status, void* stream) {
  if (!p || p->generic || p->mode_t) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  int cap = 0;
  int rc = check_geometry(R, p->E, N, L, &cap);
  if (rc != CYR_OK) return rc;
  if (R == 0) return CYR_OK;
  if (!alloc || !k || !grants || !status) return CYR_BAD_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int E = p->E;
  const size_t raw_b = ((size_t)R * 2 * E * p->elem + 255) / 256 * 256;
  const size_t mat_b = ((size_t)R * E * 8 + 255) / 256 * 256;
  unsigned char* ws = nullptr;
  if (cyr::malloc_async(reinterpret_cast<void**>(&ws), raw_b + 3 * mat_b + (size_t)R * 8, st) !=
      cudaSuccess)
    return cuda_fail(cudaGetLastError(), "cudaMallocAsync(actions)");
  void* raw = ws;
  double* b = b_out ? b_out : reinterpret_cast<double*>(ws + raw_b);
  double* caps = reinterpret_cast<double*>(ws + raw_b + mat_b);
  int64_t* demand = reinterpret_cast<int64_t*>(ws + raw_b + 2 * mat_b);
  const int prec = simt_precision(p);
  rc = cyr_launch_actor_columns(prec, p->desc, p->blob_d, alloc, k, nullptr, R, E, N, cap, raw,
                                p->sm_count, st);
  if (rc == CYR_OK)
    rc = cyr_launch_actions_head(prec, raw, alloc, k, eps, R, E, L, b, caps, demand, log_pi,
                                 status, st);
  if (rc == CYR_OK)
    rc = cyr_launch_enforce(b, caps, nullptr, demand, R, E, nullptr, nullptr, nullptr, grants,
                            nullptr, status, st);
  cudaFreeAsync(ws, st);
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

namespace {
// stop the policy's server, then wait for every launch that may still read
// the old weights (the library's streams and the caller's: device-wide, with
// every resident server told to leave first so the wait is only real work)
int quiesce_for_upload(cyr_policy* p) {
  slot_server_stop(p);
  CYR_CUDA(device_sync_quiet());
  return CYR_OK;
}


// any watched host array differs from the snapshot last published from it
bool watch_changed(const cyr_policy* p) {
  const auto& w = p->watch;
  size_t off = 0;
  for (size_t i = 0; i < w.ptr.size(); ++i) {
    if (std::memcmp(w.ptr[i], w.snap + off, w.count[i] * sizeof(double)) != 0) return true;
    off += w.count[i];
  }
  return false;
}

// snapshot the watched arrays and publish them
int watch_republish(cyr_policy* p) {
  auto& w = p->watch;
  size_t off = 0;
  for (size_t i = 0; i < w.ptr.size(); ++i) {
    std::memcpy(w.snap + off, w.ptr[i], w.count[i] * sizeof(double));
    off += w.count[i];
  }
  const int rc = quiesce_for_upload(p);
  return rc != CYR_OK ? rc : upload(p, w.snap);
}
}  // namespace

int cyr_policy_sample_device(const cyr_policy* p, const int32_t* alloc, const int32_t* k,
                             const double* eps, int32_t R, int32_t N, int32_t L, double* b_out,
                             double* log_pi, int32_t* status, void* stream) {
  if (!p || p->generic || p->mode_t) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  int cap = 0;
  int rc = check_geometry(R, p->E, N, L, &cap);
  if (rc != CYR_OK) return rc;
  if (R == 0) return CYR_OK;
  if (!alloc || !k || !b_out || !status) return CYR_BAD_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int E = p->E;
  const size_t raw_b = ((size_t)R * 2 * E * p->elem + 255) / 256 * 256;
  const size_t mat_b = ((size_t)R * E * 8 + 255) / 256 * 256;
  unsigned char* ws = nullptr;
  if (cyr::malloc_async(reinterpret_cast<void**>(&ws), raw_b + mat_b + (size_t)R * 8, st) !=
      cudaSuccess)
    return cuda_fail(cudaGetLastError(), "cudaMallocAsync(sample)");
  double* caps = reinterpret_cast<double*>(ws + raw_b);
  int64_t* demand = reinterpret_cast<int64_t*>(ws + raw_b + mat_b);
  const int prec = simt_precision(p);
  rc = cyr_launch_actor_columns(prec, p->desc, p->blob_d, alloc, k, nullptr, R, E, N, cap, ws,
                                p->sm_count, st);
  if (rc == CYR_OK)
    rc = cyr_launch_actions_head(prec, ws, alloc, k, eps, R, E, L, b_out, caps, demand, log_pi,
                                 status, st);
  cudaFreeAsync(ws, st);
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_policy_update(cyr_policy* p, const double* weights_blob) {
  if (!p || !weights_blob) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  const int rc = quiesce_for_upload(p);
  if (rc != CYR_OK) return rc;
  if (!p->watch.ptr.empty())  // an explicit publish is the new snapshot
    std::memcpy(p->watch.snap, weights_blob, p->watch.snap_n * sizeof(double));
  return upload(p, weights_blob);
}

int cyr_policy_watch(cyr_policy* p, const double* const* arrays, const int64_t* counts,
                     int32_t n) {
  if (!p || n < 0 || (n > 0 && (!arrays || !counts))) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  auto& w = p->watch;
  if (n == 0) {
    w.ptr.clear();
    w.count.clear();
    return CYR_OK;
  }
  // flatten order: W_l (out*in) then b_l (out) for every layer
  if ((size_t)n != 2 * (p->sizes.size() - 1)) return CYR_BAD_ARG;
  for (int i = 0; i < n; ++i) {
    const size_t l = (size_t)i / 2;
    const int64_t want = i % 2 == 0 ? (int64_t)p->sizes[l] * p->sizes[l + 1] : p->sizes[l + 1];
    if (counts[i] != want || !arrays[i]) return CYR_BAD_ARG;
  }
  w.ptr.assign(arrays, arrays + n);
  w.count.assign(counts, counts + n);
  if (!w.snap) {
    w.snap_n = blob_count(p);
    CYR_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w.snap), w.snap_n * sizeof(double),
                           cudaHostAllocPortable));
  }
  return watch_republish(p);
}

int cyr_policy_sync(cyr_policy* p, int32_t* changed) {
  if (!p) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  const bool c = !p->watch.ptr.empty() && watch_changed(p);
  if (changed) *changed = c ? 1 : 0;
  return c ? watch_republish(p) : CYR_OK;
}

namespace {
int load_checkpoint(cyr_policy** out, const char* path, int32_t precision, bool generic);
}

int cyr_policy_load(cyr_policy** out, const char* path, int32_t precision) {
  return load_checkpoint(out, path, precision, false);
}

int cyr_mlp_load(cyr_policy** out, const char* path, int32_t precision) {
  return load_checkpoint(out, path, precision, true);
}

namespace {
int load_checkpoint(cyr_policy** out, const char* path, int32_t precision, bool generic) {
  if (!out || !path) return CYR_BAD_ARG;
  FILE* fh = std::fopen(path, "rb");
  if (!fh) {
    g_last_error = std::string("cannot open ") + path;
    return CYR_BAD_ARG;
  }
  std::vector<unsigned char> data;
  unsigned char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof buf, fh)) > 0) data.insert(data.end(), buf, buf + got);
  std::fclose(fh);
  auto fail = [&](const char* why) {
    g_last_error = std::string(path) + ": " + why;
    return CYR_BAD_ARG;
  };
  if (data.size() < 16 || std::memcmp(data.data(), "PSIMMLP1", 8) != 0)
    return fail("not a network checkpoint");
  uint32_t version, n_sizes;
  std::memcpy(&version, data.data() + 8, 4);
  std::memcpy(&n_sizes, data.data() + 12, 4);
  if (version != 1) return fail("unsupported format version");
  if (n_sizes < 2 || n_sizes > cyr::kMaxLayers + 1 || data.size() < 16 + 4ull * n_sizes)
    return fail("bad header");
  std::vector<int32_t> sizes(n_sizes);
  for (uint32_t i = 0; i < n_sizes; ++i) {
    uint32_t v;
    std::memcpy(&v, data.data() + 16 + 4 * i, 4);
    sizes[i] = (int32_t)v;
  }
  size_t count = 0;
  for (uint32_t i = 0; i + 1 < n_sizes; ++i)
    count += (size_t)sizes[i] * sizes[i + 1] + sizes[i + 1];
  const size_t base = 16 + 4ull * n_sizes;
  if (data.size() < base + 8 * count) return fail("checkpoint truncated");
  if (data.size() > base + 8 * count) return fail("trailing bytes");
  std::vector<double> blob(count);
  std::memcpy(blob.data(), data.data() + base, 8 * count);  // little-endian host
  return policy_create_impl(out, sizes.data(), (int32_t)n_sizes, blob.data(), precision, generic);
}
}  // namespace

int cyr_policy_quiesce(cyr_policy* p) {
  if (!p) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  slot_server_stop(p);
  return CYR_OK;
}

int cyr_quiesce_all(void) {
  stop_all_servers();
  return CYR_OK;
}

int cyr_policy_destroy(cyr_policy* p) {
  if (!p) return CYR_OK;
  {
    std::lock_guard<std::recursive_mutex> lock(p->mu);
    slot_server_stop(p);
    {
      std::lock_guard<std::mutex> reg(g_srv_mu);  // nobody signals its mailbox from here on
      g_srv_policies.erase(p);
    }
    device_sync_quiet();  // no launch still reads the policy's buffers
    if (p->srv.stream) cudaStreamDestroy(p->srv.stream);
    if (p->srv.exited) cudaEventDestroy(p->srv.exited);
    if (p->srv.mb) cudaFreeHost(p->srv.mb);
    release_host_path(p);
  }
  if (p->stream) cudaStreamDestroy(p->stream);
  if (p->ev0) cudaEventDestroy(p->ev0);
  if (p->ev1) cudaEventDestroy(p->ev1);
  cudaFree(p->blob_d);
  cudaFree(p->tc_blob_d);
  cudaFree(p->wide_act_d);
  cudaFree(p->raw_stage_d);
  if (p->up_stream) cudaStreamDestroy(p->up_stream);
  if (p->watch.snap) cudaFreeHost(p->watch.snap);
  delete p;
  return CYR_OK;
}

int cyr_policy_info(const cyr_policy* p, int32_t* num_users, int32_t* n_sizes, int32_t* precision) {
  if (!p) return CYR_BAD_ARG;
  if (num_users) *num_users = p->E;
  if (n_sizes) *n_sizes = (int32_t)p->sizes.size();
  if (precision) *precision = p->precision;
  return CYR_OK;
}

int cyr_actor_forward_device(const cyr_policy* p, const int32_t* alloc, int32_t S, int32_t N,
                             int32_t cap, void* raw, void* stream) {
  if (!p || p->mode_t || (S > 0 && (!alloc || !raw)) || N <= 0 || cap < 1) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  const int rc = launch_actor_policy(p, alloc, S, N, cap, raw, static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

size_t cyr_raw_bytes(const cyr_policy* p, int32_t S, int32_t cap) {
  if (!p || S < 0 || cap < 0) return 0;
  return (size_t)S * cap * 2 * p->E * p->elem;
}

int cyr_codebook_from_raw_device(const cyr_policy* p, const void* raw, const int32_t* alloc,
                                 const double* eps, int32_t S, int32_t N, int32_t L,
                                 int32_t* codebook, double* m_hat, double* nu, double* margin,
                                 int32_t* iters, int32_t* status, void* stream) {
  if (!p) return CYR_BAD_ARG;
  int cap = 0;
  int rc = check_geometry(S, p->E, N, L, &cap);
  if (rc != CYR_OK) return rc;
  if (S > 0 && (!raw || !alloc || !codebook)) return CYR_BAD_ARG;
  rc = cyr_launch_codebook(p->precision, raw, alloc, eps, S, p->E, N, L, cap, codebook, m_hat, nu,
                           margin, iters, status, static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_codebook_device(const cyr_policy* p, const int32_t* alloc, const double* eps, int32_t S,
                        int32_t N, int32_t L, int32_t* codebook, void* raw_workspace,
                        int32_t* status, void* stream) {
  if (!p || p->mode_t) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  int cap = 0;
  int rc = check_geometry(S, p->E, N, L, &cap);
  if (rc != CYR_OK) return rc;
  if (S > 0 && S * cap <= 8) {  // latency path: K2 + K3 in one cluster launch
    rc = cyr_launch_slot_fused(p->precision, p->desc, p->blob_d, alloc, eps, S, p->E, N, L, cap,
                               codebook, nullptr, status, static_cast<cudaStream_t>(stream));
    if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
    return rc;
  }
  rc = cyr_actor_forward_device(p, alloc, S, N, cap, raw_workspace, stream);
  if (rc != CYR_OK) return rc;
  return cyr_codebook_from_raw_device(p, raw_workspace, alloc, eps, S, N, L, codebook, nullptr,
                                      nullptr, nullptr, nullptr, status, stream);
}

// ---- persistent slot server (the fused path without per-call launches) ----
// CYR_SLOT_SERVER=0 falls back to the per-call graph launch (A/B);
// CYR_SLOT_SERVER_IDLE_MS: how long an idle server keeps polling (default 20).
static bool slot_server_enabled() {
  static const bool on = [] {
    const char* e = getenv("CYR_SLOT_SERVER");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

static unsigned long long slot_server_idle_ns() {
  static const unsigned long long ns = [] {
    const char* e = getenv("CYR_SLOT_SERVER_IDLE_MS");
    const double ms = e ? atof(e) : 20.0;
    return (unsigned long long)((ms > 0.0 ? ms : 20.0) * 1e6);
  }();
  return ns;
}

// stop a running server and wait for it to leave (before anything that
// synchronises the whole device, and before the policy changes)
static void slot_server_stop(cyr_policy* p) {
  auto& sv = p->srv;
  if (!sv.running.load()) return;
  sv.mb->quit = 1u;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  cudaEventSynchronize(sv.exited);
  sv.mb->quit = 0u;
  sv.running.store(false);
}

static int slot_server_launch(cyr_policy* p, bool det, int S, int N, int L, int cap) {
  auto& sv = p->srv;
  const int rc = cyr_launch_slot_server(p->precision, p->desc, p->blob_d, det, S, p->E, N, L, cap,
                                        p->cb_d, sv.mb_dev, sv.seq, slot_server_idle_ns(),
                                        sv.stream);
  if (rc != CYR_OK) {
    if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
    return rc;
  }
  CYR_CUDA(cudaEventRecord(sv.exited, sv.stream));
  sv.running.store(true);
  return CYR_OK;
}

// One request through the server: inputs into the mailbox, bump req_seq,
// spin on done_seq.  A server that idled out just before the request is
// relaunched (it picks the pending request up: it starts from the last
// request served).  CYR_UNSUPPORTED: geometry outside the server's range.
static int slot_server_call(cyr_policy* p, const std::tuple<int, int, int, int>& key,
                            const int32_t* alloc, const double* eps, int S, int N, int L, int cap,
                            int32_t* codebook, int64_t* device_ns, bool* stale) {
  auto& sv = p->srv;
  const int E = p->E;
  if (S * (cap + 1) * E > 512 || S * E > 256 || S * cap * E > 256) return CYR_UNSUPPORTED;
  if (sv.mb == nullptr) {
    CYR_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sv.mb), sizeof(cyr::SlotMailbox),
                           cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(static_cast<void*>(sv.mb), 0, sizeof(cyr::SlotMailbox));
    CYR_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&sv.mb_dev), sv.mb, 0));
    CYR_CUDA(cudaStreamCreateWithFlags(&sv.stream, cudaStreamNonBlocking));
    CYR_CUDA(cudaEventCreateWithFlags(&sv.exited, cudaEventDisableTiming));
    std::lock_guard<std::mutex> reg(g_srv_mu);
    g_srv_policies.insert(p);
  }
  const bool det = (eps == nullptr);
  if (sv.running.load() && sv.key != key) slot_server_stop(p);
  if (sv.running.load() && cudaEventQuery(sv.exited) == cudaSuccess)
    sv.running.store(false);  // idled out (or told to leave by stop_all_servers)
  std::memcpy(sv.mb->alloc, alloc, (size_t)S * E * 4);
  if (!det) std::memcpy(sv.mb->eps, eps, (size_t)S * cap * E * 8);
  sv.mb->status = CYR_OK;
  if (!sv.running.load()) {
    const int rc = slot_server_launch(p, det, S, N, L, cap);
    if (rc != CYR_OK) return rc;
    sv.key = key;
  }
  uint32_t next = sv.seq + 1u;
  if (next == 0u) next = 1u;  // 0 means "leave" to the server
  std::atomic_thread_fence(std::memory_order_release);
  sv.mb->req_seq = next;
  host_stamp(1);
  // "check" weight sync: compare the caller's host weights with the
  // published snapshot while the cluster computes (~20 us of device work
  // hides the memcmp); a stale answer is recomputed by the caller
  if (stale) *stale = !p->watch.ptr.empty() && watch_changed(p);
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 1;; ++spin) {
    if (sv.mb->done_seq == next) break;
    if ((spin & 4095u) == 0u) {
      if (cudaEventQuery(sv.exited) == cudaSuccess && sv.mb->done_seq != next) {
        // the server left (idle timeout) without seeing this request: relaunch
        const int rc = slot_server_launch(p, det, S, N, L, cap);
        if (rc != CYR_OK) return rc;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10)) {
        slot_server_stop(p);
        g_last_error = "slot server did not answer within 10 s";
        return CYR_CUDA_ERROR;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  sv.seq = next;
  host_stamp(4);
  const int32_t code = sv.mb->status;
  if (code != CYR_OK) return code;
  std::memcpy(codebook, sv.mb->cb, (size_t)S * (cap + 1) * E * 4);
  if (device_ns) *device_ns = (int64_t)(sv.mb->t_end - sv.mb->t_start);
  return CYR_OK;
}

static int codebook_host_once(cyr_policy* p, const int32_t* alloc, const double* eps, int32_t S,
                              int32_t N, int32_t L, int32_t* codebook, int64_t* device_ns,
                              bool* stale) {
  if (stale) *stale = false;
  if (!p || p->mode_t || !alloc || !codebook) return CYR_BAD_ARG;
  int cap = 0;
  int rc = check_geometry(S, p->E, N, L, &cap);
  if (rc != CYR_OK) return rc;
  if (S == 0) return CYR_OK;
  const int E = p->E;
  // reference validation order: negative inputs (ValueError), then
  // demand > capacity (InfeasibleDemandError, enforcer.py:64)
  for (int s = 0; s < S; ++s) {
    long long total = 0;
    for (int e = 0; e < E; ++e) {
      if (alloc[(size_t)s * E + e] < 0) return CYR_BAD_ARG;
      total += alloc[(size_t)s * E + e];
    }
    if ((long long)cap * L > total) return CYR_INFEASIBLE;
  }
  rc = ensure_host_path(p, S, cap);
  if (rc != CYR_OK) return rc;
  std::memcpy(p->pin_alloc, alloc, (size_t)S * E * 4);
  const bool det = (eps == nullptr);
  if (!det) std::memcpy(p->pin_eps, eps, (size_t)S * cap * E * 8);

  const auto key = std::make_tuple(S, N, L, det ? 1 : 0);
  const bool fused = S * cap <= 8 && S * E <= 256 && S * cap * E <= 256;
  auto dev = [&](const void* host_ptr) {  // device alias of a mapped host pointer
    return reinterpret_cast<unsigned char*>(p->pin_dev) +
           (reinterpret_cast<const unsigned char*>(host_ptr) - p->pin);
  };
  *p->pin_status = CYR_OK;
  if (fused && slot_server_enabled()) {
    // latency path: the resident slot server (no launch per call)
    host_stamp(0);
    const int src = slot_server_call(p, key, alloc, eps, S, N, L, cap, codebook, device_ns, stale);
    if (src != CYR_UNSUPPORTED) return src;
  }
  if (p->srv.running.load()) slot_server_stop(p);  // the batch paths below synchronise streams
  if (fused) {
    // latency path: ONE cluster launch (K2 + K3), inputs by value in the
    // launch parameters, codebook + status written straight to mapped pages
    host_stamp(0);
    cyr::SlotInline inl;
    std::memcpy(inl.alloc, alloc, (size_t)S * E * 4);
    if (!det) std::memcpy(inl.eps, eps, (size_t)S * cap * E * 8);
    cudaStream_t st = p->stream;
    static const bool use_graph = [] {
      const char* e = getenv("CYR_SLOT_GRAPH");
      return !(e != nullptr && e[0] == '0');
    }();
    auto launch = [&](cudaStream_t s) {
      return cyr_launch_slot_fused(p->precision, p->desc, p->blob_d, nullptr, eps, S, E, N, L,
                                   cap, p->cb_d, reinterpret_cast<int32_t*>(dev(p->pin_cb)),
                                   reinterpret_cast<int32_t*>(dev(p->pin_status)), s, &inl);
    };
    if (!use_graph) {
      CYR_CUDA(cudaEventRecord(p->ev0, st));
      const int lrc = launch(st);
      if (lrc != CYR_OK) {
        if (lrc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
        return lrc;
      }
      CYR_CUDA(cudaEventRecord(p->ev1, st));
    } else {
      auto fit = p->fused.find(key);
      if (fit == p->fused.end()) {
        cyr_policy::FusedGraph fg;
        CYR_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        cudaEventRecordWithFlags(p->ev0, st, cudaEventRecordExternal);
        const int lrc = launch(st);
        cudaEventRecordWithFlags(p->ev1, st, cudaEventRecordExternal);
        CYR_CUDA(cudaStreamEndCapture(st, &fg.graph));
        if (lrc != CYR_OK) {
          cudaGraphDestroy(fg.graph);
          return lrc;
        }
        size_t n = 0;
        CYR_CUDA(cudaGraphGetNodes(fg.graph, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        CYR_CUDA(cudaGraphGetNodes(fg.graph, nodes.data(), &n));
        for (cudaGraphNode_t nd : nodes) {
          cudaGraphNodeType t;
          CYR_CUDA(cudaGraphNodeGetType(nd, &t));
          if (t == cudaGraphNodeTypeKernel) fg.node = nd;
        }
        if (!fg.node) return CYR_CUDA_ERROR;
        CYR_CUDA(cudaGraphKernelNodeGetParams(fg.node, &fg.kp));
        cudaError_t e = cudaGraphInstantiate(&fg.exec, fg.graph, 0);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate(fused)");
        fit = p->fused.emplace(key, fg).first;
      }
      // new inputs: same ActorLaunch (the node's stored copy), fresh SlotInline
      cudaKernelNodeParams kp = fit->second.kp;
      void* args[2] = {kp.kernelParams[0], &inl};
      kp.kernelParams = args;
      host_stamp(1);
      CYR_CUDA(cudaGraphExecKernelNodeSetParams(fit->second.exec, fit->second.node, &kp));
      host_stamp(2);
      CYR_CUDA(cudaGraphLaunch(fit->second.exec, st));
      host_stamp(3);
    }
    if (stale) *stale = !p->watch.ptr.empty() && watch_changed(p);  // overlaps the kernel
    CYR_CUDA(cudaEventSynchronize(p->ev1));
    host_stamp(4);
    const int32_t code = *reinterpret_cast<volatile int32_t*>(p->pin_status);
    if (code != CYR_OK) return code;
    std::memcpy(codebook, p->pin_cb, (size_t)S * (cap + 1) * E * 4);
    if (device_ns) {
      float ms = 0.f;
      CYR_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
      *device_ns = (int64_t)std::llround((double)ms * 1e6);
    }
    return CYR_OK;
  }
  auto it = p->graphs.find(key);
  if (it == p->graphs.end()) {
    cudaStream_t st = p->stream;
    CYR_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    cudaEventRecordWithFlags(p->ev0, st, cudaEventRecordExternal);
    int lrc = CYR_OK;
    {
      (void)dev;
      cudaMemcpyAsync(p->alloc_d, p->pin_alloc, (size_t)S * E * 4, cudaMemcpyHostToDevice, st);
      if (!det)
        cudaMemcpyAsync(p->eps_d, p->pin_eps, (size_t)S * cap * E * 8, cudaMemcpyHostToDevice,
                        st);
      cudaMemsetAsync(p->status_d, 0, 4, st);
      lrc = launch_actor_policy(p, p->alloc_d, S, N, cap, p->raw_d, st);
      if (lrc == CYR_OK)
        lrc = cyr_launch_codebook(p->precision, p->raw_d, p->alloc_d, det ? nullptr : p->eps_d,
                                  S, E, N, L, cap, p->cb_d, nullptr, nullptr, nullptr, nullptr,
                                  p->status_d, st);
      cudaMemcpyAsync(p->pin_cb, p->cb_d, (size_t)S * (cap + 1) * E * 4, cudaMemcpyDeviceToHost,
                      st);
      cudaMemcpyAsync(p->pin_status, p->status_d, 4, cudaMemcpyDeviceToHost, st);
    }
    cudaEventRecordWithFlags(p->ev1, st, cudaEventRecordExternal);
    cudaGraph_t graph = nullptr;
    CYR_CUDA(cudaStreamEndCapture(st, &graph));
    if (lrc != CYR_OK) {
      cudaGraphDestroy(graph);
      return lrc;
    }
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    it = p->graphs.emplace(key, exec).first;
  }
  CYR_CUDA(cudaGraphLaunch(it->second, p->stream));
  if (stale) *stale = !p->watch.ptr.empty() && watch_changed(p);  // overlaps the graph
  CYR_CUDA(cudaStreamSynchronize(p->stream));
  if (*p->pin_status != CYR_OK) return *p->pin_status;
  std::memcpy(codebook, p->pin_cb, (size_t)S * (cap + 1) * E * 4);
  if (device_ns) {
    float ms = 0.f;
    CYR_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    *device_ns = (int64_t)std::llround((double)ms * 1e6);
  }
  return CYR_OK;
}

int cyr_codebook_host(cyr_policy* p, const int32_t* alloc, const double* eps, int32_t S,
                      int32_t N, int32_t L, int32_t* codebook, int64_t* device_ns) {
  if (!p) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  bool stale = false;
  int rc = codebook_host_once(p, alloc, eps, S, N, L, codebook, device_ns, &stale);
  if (stale) {  // the watched host weights changed in place: republish and recompute
    const int r2 = watch_republish(p);
    if (r2 != CYR_OK) return r2;
    rc = codebook_host_once(p, alloc, eps, S, N, L, codebook, device_ns, nullptr);
  }
  return rc;
}

int cyr_enforce_batch_device(const double* b, const double* caps, const int64_t* demand,
                             int32_t R, int32_t E, double* m_hat, double* nu,
                             uint8_t* degenerate, int64_t* grants, double* margin,
                             int32_t* status, void* stream) {
  if (R < 0 || E < 1) return CYR_BAD_ARG;
  if (R > 0 && (!b || !caps || !demand || !grants)) return CYR_BAD_ARG;
  const int rc = cyr_launch_enforce(b, caps, nullptr, demand, R, E, m_hat, nu, degenerate, grants, margin,
                                    status, static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_kl_project_batch_device(const double* b, const double* caps, const double* demand,
                                int32_t R, int32_t E, double* m_hat, double* nu,
                                uint8_t* degenerate, int32_t* status, void* stream) {
  if (R < 0 || E < 1) return CYR_BAD_ARG;
  if (R > 0 && (!b || !caps || !demand || !m_hat)) return CYR_BAD_ARG;
  const int rc = cyr_launch_enforce(b, caps, demand, nullptr, R, E, m_hat, nu, degenerate,
                                    nullptr, nullptr, status, static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_apportion_batch_device(const double* m_hat, const double* caps, const int64_t* demand,
                                int32_t R, int32_t E, int64_t* grants, double* margin,
                                int32_t* status, void* stream) {
  if (R < 0 || E < 1) return CYR_BAD_ARG;
  if (R > 0 && (!m_hat || !caps || !demand || !grants)) return CYR_BAD_ARG;
  const int rc = cyr_launch_apportion(m_hat, caps, demand, R, E, grants, margin, status,
                                      static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int64_t cyr_tree_num_nodes(int32_t cap, int32_t M) {
  if (cap < 1 || M < 1) return 0;
  int64_t total = 0, level = 1;
  for (int t = 0; t < M; ++t) {
    level *= (cap + 1);
    total += level;
  }
  return total;
}

int32_t cyr_tree_state_stride(int32_t E) { return E < 1 ? 0 : (E + 1) / 2 * 2; }

int cyr_tree_expand_device(const int32_t* codebook, int32_t S, int32_t E, int32_t cap, int32_t M,
                           int16_t* node_state, void* stream) {
  if (S < 0 || (S > 0 && (!codebook || !node_state))) return CYR_BAD_ARG;
  const int rc = cyr_launch_tree(codebook, S, E, cap, M, node_state,
                                 sm_count_of_current_device(), static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_debug_trace(int64_t* out, int32_t n) {
  if (!out || n < 0) return CYR_BAD_ARG;
  for (int i = 0; i < n && i < 64; ++i)
    out[i] = g_trace_host ? (int64_t)g_trace_host[i] : 0;
  if (g_prof_dev != nullptr) {
    unsigned long long h[28] = {};
    cudaMemcpy(h, g_prof_dev, sizeof(h), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 28 && 36 + i < n; ++i) out[36 + i] = (int64_t)h[i];
  }
  return CYR_OK;
}

int cyr_selftest_latency(int32_t which, int32_t iters, int64_t* cycles) {
  if (!cycles || iters < 1) return CYR_BAD_ARG;
  long long* d = nullptr;
  double* sink = nullptr;
  CYR_CUDA(cudaMalloc(&d, sizeof(long long)));
  CYR_CUDA(cudaMalloc(&sink, 32 * sizeof(double)));
  int rc = cyr_launch_latency_bench(which, iters, d, sink);
  long long h = 0;
  if (rc == CYR_OK) {
    cudaError_t e = cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "latency bench copy");
  }
  cudaFree(d);
  cudaFree(sink);
  *cycles = (int64_t)h;
  return rc;
}

int cyr_selftest_shared_divisor(int64_t pairs_total, uint64_t seed, int64_t* mismatches) {
  if (!mismatches || pairs_total < 1) return CYR_BAD_ARG;
  const int sms = sm_count_of_current_device();
  const long long threads = (long long)sms * 8 * 256;
  unsigned long long* bad = nullptr;
  CYR_CUDA(cudaMalloc(&bad, sizeof(unsigned long long)));
  int rc = cudaMemset(bad, 0, sizeof(unsigned long long)) == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
  if (rc == CYR_OK)
    rc = cyr_launch_shared_divisor_check((pairs_total + threads - 1) / threads, seed, sms, bad,
                                         nullptr);
  unsigned long long h = 0;
  if (rc == CYR_OK && cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = CYR_CUDA_ERROR;
  cudaFree(bad);
  *mismatches = (int64_t)h;
  return rc;
}

int cyr_selftest_fma_peak(int32_t iters, double* tflops) {
  if (!tflops || iters < 1) return CYR_BAD_ARG;
  const int sms = sm_count_of_current_device();
  float* sink = nullptr;
  CYR_CUDA(cudaMalloc(&sink, sizeof(float)));
  cudaEvent_t a, b;
  CYR_CUDA(cudaEventCreate(&a));
  CYR_CUDA(cudaEventCreate(&b));
  int rc = cyr_launch_fma_peak(iters / 4 + 1, sms, sink, nullptr);  // warm-up (clocks up)
  float best_ms = 1e30f;
  for (int r = 0; r < 5 && rc == CYR_OK; ++r) {
    cudaEventRecord(a, nullptr);
    rc = cyr_launch_fma_peak(iters, sms, sink, nullptr);
    cudaEventRecord(b, nullptr);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    best_ms = std::min(best_ms, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  if (rc != CYR_OK) return rc;
  // threads x 8 chains x 2 lanes x 2 flops per iteration
  const double flops = (double)sms * 4 * 256 * 8 * 2 * 2 * (double)iters;
  *tflops = flops / (best_ms * 1e-3) / 1e12;
  return CYR_OK;
}

int cyr_selftest_launch(int32_t cluster, int32_t reps, int64_t* ns_per_launch) {
  if (!ns_per_launch || reps < 1) return CYR_BAD_ARG;
  cudaStream_t st;
  CYR_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CYR_CUDA(cudaEventCreate(&a));
  CYR_CUDA(cudaEventCreate(&b));
  double total = 0;
  for (int i = 0; i < reps + 5; ++i) {
    CYR_CUDA(cudaEventRecord(a, st));
    const int rc = cyr_launch_empty(cluster, st);
    if (rc != CYR_OK) return rc;
    CYR_CUDA(cudaEventRecord(b, st));
    CYR_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    CYR_CUDA(cudaEventElapsedTime(&ms, a, b));
    if (i >= 5) total += ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(st);
  *ns_per_launch = (int64_t)(total * 1e6 / reps);
  return CYR_OK;
}

// ---------------------------------------------------------------- Mode T
size_t cyr_tree_mode_t_workspace_bytes(const cyr_policy* p, int32_t S, int32_t cap, int32_t M) {
  if (!p || S < 0 || cap < 1 || M < 1) return 0;
  long long widest = 1;
  for (int t = 1; t < M; ++t) widest *= (cap + 1);  // parents of the deepest level
  const size_t raw = ((size_t)S * widest * cap * 2 * p->E * p->elem + 255) / 256 * 256;
  const long long cols = (long long)S * widest * cap;
  size_t act = wide_act_bytes(p, cols);
  if (p->precision != CYR_BF16_TC && cyr_gemm_path_applies(simt_precision(p), p->desc, cols))
    act = std::max(act, cyr_gemm_workspace_bytes(p->desc, cols));
  return raw + act;
}

int cyr_ldpc_peel_device(const int32_t* edge_var, const int32_t* edge_check, int32_t n,
                         int32_t n_checks, int32_t n_edges, const uint8_t* erased, int32_t B,
                         uint8_t* ok, void* stream) {
  if (n < 1 || n_checks < 1 || n_edges < 1 || B < 0) return CYR_BAD_ARG;
  if (B > 0 && (!edge_var || !edge_check || !erased || !ok)) return CYR_BAD_ARG;
  const int rc = cyr_launch_ldpc_peel(edge_var, edge_check, n, n_checks, n_edges, erased, nullptr,
                                      1, 0, B, ok, static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_ldpc_peel_counts_device(const int32_t* edge_var, const int32_t* edge_check, int32_t n,
                                int32_t n_checks, int32_t n_edges, const int32_t* counts,
                                int32_t M, int32_t n_sym, int32_t B, uint8_t* ok, void* stream) {
  if (n < 1 || n_checks < 1 || n_edges < 1 || B < 0 || M < 1 || n_sym < 0 || n_sym > n)
    return CYR_BAD_ARG;
  if (B > 0 && (!edge_var || !edge_check || !counts || !ok)) return CYR_BAD_ARG;
  const int rc = cyr_launch_ldpc_peel(edge_var, edge_check, n, n_checks, n_edges, nullptr, counts,
                                      M, n_sym, B, ok, static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_pf_schedule_device(double* avg_tput, const double* inst_rate, int32_t C, int32_t E,
                           double beta, int32_t num_rbs, int32_t rb_size, int32_t* alloc,
                           int32_t* status, void* stream) {
  if (C < 0 || E < 1 || num_rbs < 0 || rb_size < 1 || !(beta >= 0.0 && beta <= 1.0))
    return CYR_BAD_ARG;
  if (C > 0 && (!avg_tput || !inst_rate || !alloc || !status)) return CYR_BAD_ARG;
  if ((long long)num_rbs * rb_size > (1ll << 30)) return CYR_BAD_ARG;
  const int rc = cyr_launch_pf_schedule(avg_tput, inst_rate, C, E, beta, num_rbs, rb_size, alloc,
                                        status, static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_tree_score_device(const int32_t* codebook, const int32_t* alloc, const double* margin,
                          const double* prob, int32_t S, int32_t E, int32_t cap, int32_t M,
                          int32_t N, int16_t* node_state, uint32_t* leaf_ok, double* expect,
                          void* stream) {
  if (S < 0 || E < 1 || cap < 1 || M < 1) return CYR_BAD_ARG;
  if (S > 0 && (!codebook || !alloc || !margin || !prob || !node_state)) return CYR_BAD_ARG;
  if (M * N > 32767) return CYR_UNSUPPORTED;  // int16 cumulative punctures
  const int rc = cyr_launch_tree_score(codebook, alloc, margin, prob, S, E, cap, M, N, node_state,
                                       leaf_ok, expect, sm_count_of_current_device(),
                                       static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_tree_leaf_score_states_device(const int16_t* node_state, int64_t nodes_per_slot,
                                      int32_t S, int32_t E, int32_t cap, int32_t M,
                                      int64_t first, int64_t count, const int32_t* alloc,
                                      const double* margin, const double* prob, int32_t N,
                                      uint32_t* leaf_ok, double* expect, void* stream) {
  if (S < 0 || E < 1 || E > 32 || cap < 1 || M < 1 || M > 10 || N <= 0) return CYR_BAD_ARG;
  long long leaves = 1;
  for (int t = 0; t < M; ++t) leaves *= cap + 1;
  if (first < 0 || count < 0 || first + count > leaves) return CYR_BAD_ARG;
  if (nodes_per_slot != cyr_tree_num_nodes(cap, M)) return CYR_BAD_ARG;
  if (S == 0 || count == 0) return CYR_OK;
  if (!node_state || !alloc || !margin || !prob || !expect) return CYR_BAD_ARG;
  const int epad = cyr_tree_state_stride(E);
  const long long leaf0 = nodes_per_slot - leaves;  // level M is the last run of BFS order
  const int rc = cyr_launch_leaf_states_score(
      node_state + (leaf0 + first) * epad, nodes_per_slot * epad, S, E, epad, first, count, cap,
      M, alloc, margin, prob, N, leaf_ok, expect, static_cast<cudaStream_t>(stream));
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

int cyr_tree_mode_t_device(const cyr_policy* p, const int32_t* alloc, const int32_t* mcs,
                           const double* eps, int32_t S, int32_t N, int32_t L, int32_t M,
                           double mcs_scale, int16_t* node_state, void* workspace,
                           int32_t* status, void* stream) {
  return cyr_tree_mode_t_shard_device(p, alloc, mcs, eps, S, N, L, M, mcs_scale, 0, 0, 1,
                                      node_state, workspace, status, stream);
}

int cyr_tree_mode_t_shard_device(const cyr_policy* p, const int32_t* alloc, const int32_t* mcs,
                                 const double* eps, int32_t S, int32_t N, int32_t L, int32_t M,
                                 double mcs_scale, int32_t shard_level, int64_t first,
                                 int64_t count, int16_t* node_state, void* workspace,
                                 int32_t* status, void* stream) {
  if (!p || !p->mode_t) return CYR_BAD_ARG;
  std::lock_guard<std::recursive_mutex> lock(p->mu);
  int cap = 0;
  int rc = check_geometry(S, p->E, N, L, &cap);
  if (rc != CYR_OK) return rc;
  if (M < 1 || M > 10 || mcs_scale <= 0.0) return CYR_BAD_ARG;
  const int R = cap + 1;
  if (shard_level < 0 || shard_level > M) return CYR_BAD_ARG;
  long long width = 1;  // nodes of level shard_level
  for (int t = 0; t < shard_level; ++t) width *= R;
  if (first < 0 || count < 0 || first + count > width) return CYR_BAD_ARG;
  if (S == 0) return CYR_OK;  // count == 0 still builds the replicated levels
  if (!alloc || !mcs || !node_state || !workspace) return CYR_BAD_ARG;
  const int epad = cyr_tree_state_stride(p->E);
  const long long nodes = cyr_tree_num_nodes(cap, M);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // level tau's parents (level tau-1): all of them while tau-1 < shard_level
  // (replicated on every shard), else the descendants of level-shard_level
  // nodes [first, first + count): a contiguous range in BFS order
  long long level_off = 0, prev_off = -1, level_size = 1;  // level tau-1: offset, size
  for (int tau = 1; tau <= M; ++tau) {
    long long base = 0, parents = level_size;
    if (tau - 1 >= shard_level) {
      long long span = 1;
      for (int t = shard_level; t < tau - 1; ++t) span *= R;
      base = first * span;
      parents = count * span;
      if (parents == 0) break;
    }
    const long long par_off = prev_off < 0 ? -1 : prev_off + base;
    // K2: the actor on every (parent, branch) column of this level
    const long long cols = (long long)S * parents * cap;
    if (use_tc_fused(p) && cols >= kTcMinCols) {
      rc = cyr_launch_actor_tc_fused(p->desc, p->tc_blob_d, p->tc_off, p->tc_npad,
                                     static_cast<const float*>(p->blob_d), alloc, S, p->E, N, cap,
                                     static_cast<float*>(workspace), 1, mcs, node_state, M, tau,
                                     (int)parents, nodes, par_off, epad, mcs_scale, p->sm_count,
                                     st, (int)base);
    } else if (p->tc_wide || (p->tc_layers && cols >= kTcLayerCols)) {
      long long widest = 1;
      for (int t = 1; t < M; ++t) widest *= R;
      unsigned char* act = static_cast<unsigned char*>(workspace) +
                           ((size_t)S * widest * cap * 2 * p->E * p->elem + 255) / 256 * 256;
      rc = launch_actor_wide(p, alloc, S, N, cap, static_cast<float*>(workspace), act, cols, 1, mcs,
                             node_state, M, tau, (int)parents, nodes, par_off, epad, mcs_scale, st,
                             (int)base);
    } else if (p->tc_ok && cols >= kTcMinCols)
      rc = cyr_launch_actor_tc(p->desc, p->tc_blob_d, p->tc_off, p->tc_npad,
                               static_cast<const float*>(p->blob_d), alloc, S, p->E, N, cap,
                               static_cast<float*>(workspace), 1, mcs, node_state, M, tau,
                               (int)parents, nodes, par_off, epad, mcs_scale, st, (int)base);
    else {
      long long widest = 1;
      for (int t = 1; t < M; ++t) widest *= R;
      void* gemm_ws = static_cast<unsigned char*>(workspace) +
                      ((size_t)S * widest * cap * 2 * p->E * p->elem + 255) / 256 * 256;
      rc = cyr_launch_actor_mode_t(simt_precision(p), p->desc, p->blob_d, alloc, mcs, node_state,
                                   S, p->E, N, cap, M, tau, (int)parents, nodes, par_off, epad,
                                   mcs_scale, workspace, p->sm_count, st, (int)base, gemm_ws);
    }
    if (rc != CYR_OK) break;
    // K3: one coupled enforcement per parent; writes the children's states
    const long long level_tau_off = prev_off < 0 ? 0 : prev_off + level_size;
    rc = cyr_launch_tree_level(simt_precision(p), workspace, alloc, eps, node_state, S, p->E, L, cap,
                               (int)parents, epad, nodes, par_off, level_tau_off + base * R, status,
                               st);
    if (rc != CYR_OK) break;
    prev_off = level_tau_off;
    level_size *= R;
  }
  (void)level_off;
  if (rc == CYR_CUDA_ERROR) g_last_error = cudaGetErrorString(cudaGetLastError());
  return rc;
}

}  // extern "C"
