// codebook.cu — K3 kernels: batch codebook (one CTA per slot), standalone
// enforcer (one coupled call per CTA) and standalone Huntington-Hill.
// Device code lives in projection.cuh.
#include "projection.cuh"
#include "projection_lane.cuh"

namespace cyr {

// the lane kernels' seat-priority divisor table (projection_lane.cuh), built
// once per device before the first lane launch
inline int ensure_seat_table(cudaStream_t stream) {
  (void)stream;  // built on a private stream: legal while the caller's stream is being captured
  static AttrCache built;
  const bool ok = ensure_func_attr(built, 0, [&] {
    cudaStream_t st = nullptr;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return false;
    seat_table_kernel<<<1, 256, 0, st>>>();
    const bool done = cudaStreamSynchronize(st) == cudaSuccess;
    cudaStreamDestroy(st);
    return done;
  });
  return ok ? CYR_OK : CYR_CUDA_ERROR;
}

// ------------------------------------------------------------ codebook K3
// A CTA holds `spc` whole slots (<= 32 rows); 8 warps stride over the rows
// in the per-row phases and warp 0 runs every slot's coupled loop at once.
template <typename RawT, int KE = 0>
__global__ void __launch_bounds__(256, 4) codebook_kernel(
    const RawT* __restrict__ raw, const int32_t* __restrict__ alloc,
    const double* __restrict__ eps, int S, int spc, int E, int L, int cap,
    int32_t* __restrict__ cb, double* __restrict__ m_out, double* __restrict__ nu_out,
    double* __restrict__ margin_out, int32_t* __restrict__ iters_out,
    int32_t* __restrict__ status) {
  __shared__ RowScratch sc;
  const long long s0 = (long long)blockIdx.x * spc;
  const int slots = (int)min((long long)spc, S - s0);
  const long long row0 = s0 * cap;
  codebook_rows<RawT, KE>(raw + row0 * 2 * E, alloc, eps, row0, slots * cap, cap, E, L, cb, m_out,
                          nu_out, margin_out, iters_out, status, sc);
}

// Batch K3, one lane per row (projection_lane.cuh): each warp holds
// 32 / cap whole slots; 4 warps per CTA, no CTA barrier.
constexpr int kLaneWarps = 4;
#ifndef CYR_LANE_MINB
#define CYR_LANE_MINB 7
#endif
constexpr int kLaneMinBlocks = CYR_LANE_MINB;  // <= 72 registers: 28 warps per SM at E = 10 (5 / 6 / 7 / 8: 1,004 / 983 / 972 / 988 us, deepest cfg2 level)

template <typename RawT, int KE = 0>
__global__ void __launch_bounds__(32 * kLaneWarps) codebook_lane_kernel(
    const RawT* __restrict__ raw, const int32_t* __restrict__ alloc,
    const double* __restrict__ eps, int S, int E, int L, int cap, int32_t* __restrict__ cb,
    double* __restrict__ m_out, double* __restrict__ nu_out, double* __restrict__ margin_out,
    int32_t* __restrict__ iters_out, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char lane_smem[];
  const int w = threadIdx.x >> 5;
  const int gpw = 32 / cap;
  const long long s0 = ((long long)blockIdx.x * kLaneWarps + w) * gpw;
  if (s0 >= S) return;
  const int slots = (int)min((long long)gpw, S - s0);
  const long long row0 = s0 * cap;
  const SlotIO io{alloc, eps, cb, m_out, nu_out, margin_out, iters_out, E, cap};
  codebook_rows_lane<RawT, SlotIO, KE>(raw + row0 * 2 * E, row0, slots * cap, cap, E, L, io,
                                       status, lane_smem + (size_t)w * lane_scratch_bytes(E));
}

// ------------------------------------------------------------ Mode-T level
// One CTA per parent node of level tau-1, one warp per branch k: the
// parent's cap rows are one coupled enforcement call (a per-node
// build_codebook, engine.py:97-116, with node-state actor inputs); the
// grants become the children's states cum_parent + g (k = 0: cum_parent).
struct TreeIO {
  const int32_t* alloc;
  const double* eps;  // [S][cap][E]: the slot's branch-k noise, shared by its nodes
  int16_t* node;
  int E, cap, epad, parents;
  long long nodes_per_slot, parent_off, child_off;
  unsigned long long* prof;  // CYR_TRACE=1: lane-mapping phase profile, or null
  __device__ const int32_t* alloc_row(long long group) const {
    return alloc + (group / parents) * E;
  }
  __device__ const double* eps_row(long long, long long group, int j) const {
    return eps ? eps + ((group / parents) * cap + (j - 1)) * E : nullptr;
  }
  __device__ void emit(long long, long long group, int j, int lane, int g, double, double, double,
                       int) const {
    const long long s = group / parents, q = group % parents;
    const long long base = s * nodes_per_slot;
    int cum = 0;
    if (lane < E && parent_off >= 0) cum = node[(base + parent_off + q) * epad + lane];
    const long long first = (base + child_off + q * (cap + 1)) * epad;
    if (lane < epad) {
      node[first + (long long)j * epad + lane] = (int16_t)(lane < E ? cum + g : 0);
      if (j == 1) node[first + lane] = (int16_t)(lane < E ? cum : 0);
    }
  }
  // one lane = one row: child j's record (and child 0's for j == 1), one
  // 4-byte word (two users) at a time; records are epad = roundup(E, 2) lanes
  __device__ void emit_lane(long long, long long group, int j, const int* hT, int, const double*,
                            double, double, int) const {
    const long long s = group / parents, q = group % parents;
    const long long base = s * nodes_per_slot;
    const uint32_t* par =
        parent_off >= 0 ? reinterpret_cast<const uint32_t*>(node + (base + parent_off + q) * epad)
                        : nullptr;
    uint32_t* first = reinterpret_cast<uint32_t*>(node + (base + child_off + q * (cap + 1)) * epad);
    const int W = epad / 2;
    for (int w = 0; w < W; ++w) {
      const uint32_t pv = par ? par[w] : 0u;
      const int e = 2 * w;
      const int lo = (int16_t)(pv & 0xffffu), hi = (int16_t)(pv >> 16);
      const int v0 = lo + hT[e * 32];
      const int v1 = e + 1 < E ? hi + hT[(e + 1) * 32] : 0;
      first[(long long)j * W + w] = (uint32_t)(uint16_t)v0 | ((uint32_t)(uint16_t)v1 << 16);
      if (j == 1) first[w] = pv;
    }
  }
};

// K3 of one Mode-T level, one lane per row: each warp holds 32 / cap
// parents (one coupled call of cap rows each).
template <typename RawT, int KE = 0>
__global__ void __launch_bounds__(32 * kLaneWarps, kLaneMinBlocks) tree_level_kernel(const RawT* __restrict__ raw,
                                                                  TreeIO io, long long groups,
                                                                  int L,
                                                                  int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char lane_smem[];
  const int w = threadIdx.x >> 5;
  const int gpw = 32 / io.cap;
  const long long g0 = ((long long)blockIdx.x * kLaneWarps + w) * gpw;
  if (g0 >= groups) return;
  const int n = (int)min((long long)gpw, groups - g0);
  const long long row0 = g0 * io.cap;
  codebook_rows_lane<RawT, TreeIO, KE>(raw + row0 * 2 * io.E, row0, n * io.cap, io.cap, io.E, L,
                                       io, status, lane_smem + (size_t)w * lane_scratch_bytes(io.E),
                                       io.prof);
}

// K3 of a SMALL Mode-T level (few rows: the lane mapping would leave the
// machine empty and serialise E divisions per lane): one warp per row, lane
// = eMBB user, 32 / cap parents per CTA (codebook_rows_io, the latency
// path's mapping).
template <typename RawT, int KE = 0>
__global__ void __launch_bounds__(1024) tree_level_warp_kernel(const RawT* __restrict__ raw,
                                                             TreeIO io, long long groups, int L,
                                                             int32_t* __restrict__ status) {
  __shared__ RowScratch sc;
  const int gpc = 32 / io.cap;
  const long long g0 = (long long)blockIdx.x * gpc;
  const int n = (int)min((long long)gpc, groups - g0);
  const long long row0 = g0 * io.cap;
  codebook_rows_io<RawT, TreeIO, KE>(raw + row0 * 2 * io.E, row0, n * io.cap, io.cap, io.E, L, io,
                                 status, sc);
}

// ------------------------------------------------------- standalone enforcer
// One CTA = one coupled call of up to 256 rows; warps stride over rows in
// phases 1 and 3 (re-reading b and caps, which stay in L1), warp 0 runs the
// coupled loop with 8 rows per lane.
__device__ __forceinline__ Row load_row(const double* b, const double* caps, const double* demand_f,
                                        const int64_t* demand, int r, int E) {
  const int lane = threadIdx.x & 31;
  const bool in = lane < E;
  Row row;
  row.valid = true;
  row.b = in ? b[(long long)r * E + lane] : 0.0;
  row.c = in ? caps[(long long)r * E + lane] : 0.0;
  row.d = demand_f ? demand_f[r] : (double)demand[r];
  return row;
}

__global__ void __launch_bounds__(512) enforce_kernel(
    const double* __restrict__ b, const double* __restrict__ caps,
    const double* __restrict__ demand_f, const int64_t* __restrict__ demand, int R, int E,
    double* __restrict__ m_out, double* __restrict__ nu_out, uint8_t* __restrict__ degen_out,
    int64_t* __restrict__ grants, double* __restrict__ margin_out, int32_t* __restrict__ status) {
  const int nw = blockDim.x >> 5;
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool in = lane < E;
  __shared__ double s_lo[256], s_hi[256];
  __shared__ long long s_t[256];
  __shared__ int s_bis[256];
  // phase 1 (warp per row): validation, bracket, exact fill threshold
  for (int r = w; r < R; r += nw) {
    Row row = load_row(b, caps, demand_f, demand, r, E);
    const bool neg = __any_sync(kFull, row.b < 0.0 || row.c < 0.0) || row.d < 0.0;
    const double capsum = np_row_sum(row.c, E);
    if (lane == 0) {
      if (neg) set_status(status, CYR_BAD_ARG);
      else if (demand_f ? row.d > __dadd_rn(capsum, 1e-9) : row.d > capsum)
        set_status(status, CYR_INFEASIBLE);  // enforcer.py:64 / :138
    }
    kl_setup(row, E);
    long long thr = 0;
    if (row.bis) thr = fill_threshold(row, E, water_level(row, E));
    if (lane == 0) {
      s_lo[r] = row.lo;
      s_hi[r] = row.hi;
      s_t[r] = thr;
      s_bis[r] = row.bis;
    }
  }
  __syncthreads();
  // phase 2 (warp 0, lanes = rows): the coupled loop of the whole call
  if (w == 0) {
    double lo[8], hi[8];
    long long tt[8];
    bool bis[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = lane + 32 * k;
      const bool ok = r < R;
      lo[k] = ok ? s_lo[r] : 0.0;
      hi[k] = ok ? s_hi[r] : 0.0;
      tt[k] = ok ? s_t[r] : 0;
      bis[k] = ok && s_bis[r] != 0;
    }
    coupled_bisection<8>(lo, hi, tt, bis);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = lane + 32 * k;
      if (r < R) {
        s_lo[r] = lo[k];
        s_hi[r] = hi[k];
      }
    }
  }
  __syncthreads();
  // phase 3 (warp per row): m_hat, nu, Huntington-Hill
  for (int r = w; r < R; r += nw) {
    Row row = load_row(b, caps, demand_f, demand, r, E);
    kl_setup(row, E);
    row.lo = s_lo[r];
    row.hi = s_hi[r];
    double m, nu;
    kl_finish(row, E, m, nu);
    double margin = CUDART_INF;
    int g = 0;
    if (grants) g = hh_row(m, row.c, E, demand[r], margin);  // warp-uniform
    if (in) {
      if (m_out) m_out[(long long)r * E + lane] = m;
      if (grants) grants[(long long)r * E + lane] = g;
    }
    if (lane == 0) {
      if (nu_out) nu_out[r] = nu;
      if (degen_out) degen_out[r] = row.degen ? 1 : 0;
      if (margin_out) margin_out[r] = margin;
    }
  }
}

// ------------------------------------------ standalone enforcer, any R rows
// A coupled call of more rows than one CTA holds (sac.critic_targets
// enforces H*(M-1) = 1,536 rows in one call, sac.py:202-205).  Each row's
// bracket evolves independently (enforcer.py:94-97 update every bisecting
// row every step); only the STOP iteration is shared: the loop ends at the
// first t with every row converged (enforcer.py:90-92).  A row stays
// converged once it is (the bracket width at least halves each step while
// the tolerance 1e-13*hi moves by < 1 ulp-of-width), so
// t* = max over rows of the row's own first converged step.  Pass 1 finds
// each row's threshold and first converged step (atomicMax -> t*); pass 2
// replays t* steps per row, CHECKS that the row is converged there (status
// CYR_INTERNAL otherwise: the result would not be the reference's), then
// finishes m_hat / nu and Huntington-Hill like enforce_kernel.
__device__ __forceinline__ bool bracket_converged(double lo, double hi) {
  return __dsub_rn(hi, lo) <= __dmul_rn(kRelWidth, hi);  // enforcer.py:91
}
__device__ __forceinline__ void bracket_step(double& lo, double& hi, double& sl, double& sh,
                                             long long T) {
  const double mid = __dmul_rn(sl, sh);  // enforcer.py:94
  const double root = __dsqrt_rn(mid);
  if (__double_as_longlong(mid) <= T) {  // fill >= demand (exact threshold, §4.3)
    lo = mid;
    sl = root;
  } else {
    hi = mid;
    sh = root;
  }
}

__global__ void __launch_bounds__(256) enforce_wide_setup_kernel(
    const double* __restrict__ b, const double* __restrict__ caps,
    const double* __restrict__ demand_f, const int64_t* __restrict__ demand, int R, int E,
    long long* __restrict__ thr_out, int* __restrict__ stop, int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  int my_stop = 0;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += nw) {
    Row row = load_row(b, caps, demand_f, demand, r, E);
    const bool neg = __any_sync(kFull, row.b < 0.0 || row.c < 0.0) || row.d < 0.0;
    const double capsum = np_row_sum(row.c, E);
    if (lane == 0) {
      if (neg) set_status(status, CYR_BAD_ARG);
      else if (demand_f ? row.d > __dadd_rn(capsum, 1e-9) : row.d > capsum)
        set_status(status, CYR_INFEASIBLE);
    }
    kl_setup(row, E);
    long long thr = 0;
    if (row.bis) {
      thr = fill_threshold(row, E, water_level(row, E));
      double lo = row.lo, hi = row.hi, sl = __dsqrt_rn(lo), sh = __dsqrt_rn(hi);
      int t = 0;
      for (; t < kMaxIters && !bracket_converged(lo, hi); ++t) bracket_step(lo, hi, sl, sh, thr);
      my_stop = max(my_stop, t);
    }
    if (lane == 0) thr_out[r] = thr;
  }
  if (lane == 0 && my_stop > 0) atomicMax(stop, my_stop);
}

__global__ void __launch_bounds__(256) enforce_wide_finish_kernel(
    const double* __restrict__ b, const double* __restrict__ caps,
    const double* __restrict__ demand_f, const int64_t* __restrict__ demand, int R, int E,
    const long long* __restrict__ thr_in, const int* __restrict__ stop,
    double* __restrict__ m_out, double* __restrict__ nu_out, uint8_t* __restrict__ degen_out,
    int64_t* __restrict__ grants, double* __restrict__ margin_out, int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const bool in = lane < E;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int t_stop = *stop;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += nw) {
    Row row = load_row(b, caps, demand_f, demand, r, E);
    kl_setup(row, E);
    if (row.bis) {
      const long long thr = thr_in[r];
      double lo = row.lo, hi = row.hi, sl = __dsqrt_rn(lo), sh = __dsqrt_rn(hi);
      for (int t = 0; t < t_stop; ++t) bracket_step(lo, hi, sl, sh, thr);
      if (t_stop < kMaxIters && !bracket_converged(lo, hi) && lane == 0)
        set_status(status, CYR_INTERNAL);
      row.lo = lo;
      row.hi = hi;
    }
    double m, nu;
    kl_finish(row, E, m, nu);
    double margin = CUDART_INF;
    int g = 0;
    if (grants) g = hh_row(m, row.c, E, demand[r], margin);  // warp-uniform
    if (in) {
      if (m_out) m_out[(long long)r * E + lane] = m;
      if (grants) grants[(long long)r * E + lane] = g;
    }
    if (lane == 0) {
      if (nu_out) nu_out[r] = nu;
      if (degen_out) degen_out[r] = row.degen ? 1 : 0;
      if (margin_out) margin_out[r] = margin;
    }
  }
}

// ------------------------------------------------- SAC branch actions head
// sac.critic_targets' sampling block (sac.py:193-203) for R columns with
// their own allocation row and arrival count k (warp per row, lane = user):
// split_head (neural.py:144-150), sample_squashed with its log-density
// (neural.py:153-165: a = tanh(mu + sigma*eps), log pi = sum over users, in
// user order, of -log sigma - log(2 pi)/2 - eps^2/2 - log(1 - a^2 + 1e-6)),
// action_to_scs (neural.py:181-183), and the enforcement inputs: caps = the
// row's allocation, demand = k*L (sac.py:202-204).  eps == null: the
// deterministic mean tanh(mu), log pi = 0.
constexpr double kHalfLog2Pi = 0.9189385332046727;  // 0.5 * np.log(2.0 * np.pi)
constexpr double kSquashEps = 1e-6;                 // neural.py:17

template <typename RawT>
__global__ void __launch_bounds__(256) actions_head_kernel(
    const RawT* __restrict__ raw, const int32_t* __restrict__ alloc,
    const int32_t* __restrict__ kcol, const double* __restrict__ eps, int R, int E, int L,
    double* __restrict__ b_out, double* __restrict__ caps_out, int64_t* __restrict__ demand_out,
    double* __restrict__ log_pi, int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= R) return;  // warp-uniform
  const bool in = lane < E;
  const int k = kcol[r];
  if (lane == 0 && k < 1) set_status(status, CYR_BAD_ARG);
  double lp = 0.0;
  if (in) {
    const double n = (double)alloc[(long long)r * E + lane];
    const double mu = (double)raw[(long long)r * 2 * E + lane];
    const double ls =
        fmin(fmax((double)raw[(long long)r * 2 * E + E + lane], kLogSigmaMin), kLogSigmaMax);
    double a;
    if (eps != nullptr) {
      const double e = eps[(long long)r * E + lane];
      a = tanh(__dadd_rn(mu, __dmul_rn(exp(ls), e)));
      const double t = __dsub_rn(__dsub_rn(-ls, kHalfLog2Pi), __dmul_rn(0.5, __dmul_rn(e, e)));
      lp = __dsub_rn(t, log(__dadd_rn(__dsub_rn(1.0, __dmul_rn(a, a)), kSquashEps)));
    } else {
      a = tanh(mu);
    }
    b_out[(long long)r * E + lane] = __dmul_rn(__dmul_rn(__dadd_rn(a, 1.0), 0.5), n);
    caps_out[(long long)r * E + lane] = n;
  }
  double acc = shfl_d(lp, 0);  // numpy's axis-0 sum: user order, sequential
  for (int e = 1; e < E; ++e) acc = __dadd_rn(acc, shfl_d(lp, e));
  if (lane == 0) {
    demand_out[r] = (int64_t)k * L;
    if (log_pi) log_pi[r] = eps ? acc : 0.0;
  }
}

// ------------------------------------------------- standalone Huntington-Hill
// apportion_batch alone (enforcer.py:118-165): rows are independent, one
// warp per row, any number of rows.
__global__ void __launch_bounds__(256) apportion_kernel(
    const double* __restrict__ m_hat, const double* __restrict__ caps,
    const int64_t* __restrict__ demand, int R, int E, int64_t* __restrict__ grants,
    double* __restrict__ margin_out, int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;  // warp-uniform
  const bool in = lane < E;
  const double m = in ? m_hat[(long long)r * E + lane] : 0.0;
  const double c = in ? caps[(long long)r * E + lane] : 0.0;
  const long long want = demand[r];
  const double capsum = np_row_sum(c, E);
  if (lane == 0) {
    if (want < 0) set_status(status, CYR_BAD_ARG);
    else if ((double)want > capsum) set_status(status, CYR_INFEASIBLE);
  }
  double margin;
  const int g = hh_row(m, c, E, want, margin);
  if (in) grants[(long long)r * E + lane] = g;
  if (lane == 0 && margin_out) margin_out[r] = margin;
}

// ------------------------------------------------- latency microbenchmark
// Cycles per dependent step of the fp64 building blocks of the latency path
// (one warp, clock64): 0 DFMA, 1 DMUL, 2-3 __dsqrt_rn, 4 __ddiv_rn,
// 5 FFMA, 6 coupled-loop body, 7 shfl.bfly.b32, 8 __all_sync, 9 MUFU.RSQ64H.
template <int W>
__global__ void latency_bench_kernel(int iters, long long* cycles, double* sink) {
  constexpr int which = W;
  double x = 1.0000001 + threadIdx.x * 1e-9, y = 0.9999999, z = 1e-3;
  float f = 1.0001f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    switch (W) {
      case 0: x = __fma_rn(x, y, z); break;
      case 1: x = __dmul_rn(x, y); break;
      case 2: x = __dsqrt_rn(x) * 1.0000001; break;
      case 3: x = __dsqrt_rn(x) + 1.0; break;
      case 4: x = __ddiv_rn(y, x) + 1.0; break;
      case 5: f = __fmaf_rn(f, 0.9999f, 1e-4f); break;
      case 6: {
        const double mid = __dmul_rn(x, y);
        const double root = __dsqrt_rn(mid);
        const bool up = __double_as_longlong(mid) <= 0x3ff0000000000000ll;
        x = up ? root : x;
        y = up ? y : root;
        if (__all_sync(kFull, __dsub_rn(y, x) <= 1e-300)) z += 1.0;
        break;
      }
      case 7: f = __int_as_float(__shfl_xor_sync(kFull, __float_as_int(f), 1)) + 1.0f; break;
      case 8: z += __all_sync(kFull, x > 0.0) ? 1.0 : 0.0; x = x + z * 1e-300; break;
      case 10: {  // the real coupled loop: ~45 steps per call
        double lo[1] = {0.5 + threadIdx.x * 1e-6 + i * 1e-9}, hi[1] = {2.0};
        const long long t[1] = {0x3ff3c0ca4283de1bll};  // 1.2345
        const bool b[1] = {threadIdx.x < 4};
        z += coupled_bisection<1>(lo, hi, t, b, 4) + lo[0];
        break;
      }
      case 9: {
        double r;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        x = r + 1.0;
        break;
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cycles = t1 - t0;
  sink[threadIdx.x] = x + y + z + f;
}

}  // namespace cyr

int cyr_launch_actions_head(int precision, const void* raw, const int32_t* alloc,
                            const int32_t* kcol, const double* eps, int R, int E, int L,
                            double* b, double* caps, int64_t* demand, double* log_pi,
                            int32_t* status, cudaStream_t stream) {
  if (R <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers) return CYR_UNSUPPORTED;
  const int blocks = (R + 7) / 8;
  if (precision == CYR_FP64)
    cyr::actions_head_kernel<double><<<blocks, 256, 0, stream>>>(
        static_cast<const double*>(raw), alloc, kcol, eps, R, E, L, b, caps, demand, log_pi,
        status);
  else
    cyr::actions_head_kernel<float><<<blocks, 256, 0, stream>>>(
        static_cast<const float*>(raw), alloc, kcol, eps, R, E, L, b, caps, demand, log_pi,
        status);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

int cyr_launch_apportion(const double* m_hat, const double* caps, const int64_t* demand, int R,
                         int E, int64_t* grants, double* margin, int32_t* status,
                         cudaStream_t stream) {
  if (R <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers) return CYR_UNSUPPORTED;
  cyr::apportion_kernel<<<(R + 7) / 8, 256, 0, stream>>>(m_hat, caps, demand, R, E, grants,
                                                          margin, status);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

int cyr_launch_codebook(int precision, const void* raw, const int32_t* alloc, const double* eps,
                        int S, int E, int N, int L, int cap, int32_t* codebook, double* m_hat,
                        double* nu, double* margin, int32_t* iters, int32_t* status,
                        cudaStream_t stream) {
  (void)N;
  if (S <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers || cap < 1 || cap > 16) return CYR_UNSUPPORTED;
  if (S >= 1184) {  // throughput: one lane per row, 32 / cap slots per warp
    if (cyr::ensure_seat_table(stream) != CYR_OK) return CYR_CUDA_ERROR;
    const int per_cta = cyr::kLaneWarps * (32 / cap);
    const dim3 grid((S + per_cta - 1) / per_cta), block(32 * cyr::kLaneWarps);
    const size_t smem = cyr::kLaneWarps * cyr::lane_scratch_bytes(E);
    if (precision == CYR_FP64) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(cyr::codebook_lane_kernel<double>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cyr::codebook_lane_kernel<double><<<grid, block, smem, stream>>>(
          static_cast<const double*>(raw), alloc, eps, S, E, L, cap, codebook, m_hat, nu, margin,
          iters, status);
    } else {
      auto kern = E == 10 ? cyr::codebook_lane_kernel<float, 10> : cyr::codebook_lane_kernel<float, 0>;
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<grid, block, smem, stream>>>(static_cast<const float*>(raw), alloc, eps, S, E, L, cap,
                                          codebook, m_hat, nu, margin, iters, status);
    }
    return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
  }
  // small batches: one slot per CTA (latency)
  const int spc = 1;
  const dim3 grid((S + spc - 1) / spc), block(S < 1184 ? 32 * cap : 256);
#ifndef CYR_WARP_SPECIALISE
#define CYR_WARP_SPECIALISE 1
#endif
  const bool e10 = CYR_WARP_SPECIALISE && E == 10;  // cfg2 / the bench geometry
  if (precision == CYR_FP64) {
    auto kern = e10 ? cyr::codebook_kernel<double, 10> : cyr::codebook_kernel<double, 0>;
    kern<<<grid, block, 0, stream>>>(static_cast<const double*>(raw), alloc, eps, S, spc, E, L,
                                     cap, codebook, m_hat, nu, margin, iters, status);
  } else {
    auto kern = e10 ? cyr::codebook_kernel<float, 10> : cyr::codebook_kernel<float, 0>;
    kern<<<grid, block, 0, stream>>>(static_cast<const float*>(raw), alloc, eps, S, spc, E, L,
                                     cap, codebook, m_hat, nu, margin, iters, status);
  }
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

// rows of one coupled call that the single-CTA enforce_kernel holds
constexpr int kOneCtaRows = 256;

int cyr_launch_enforce(const double* b, const double* caps, const double* demand_f,
                       const int64_t* demand, int R, int E,
                       double* m_hat, double* nu, uint8_t* degenerate, int64_t* grants,
                       double* margin, int32_t* status, cudaStream_t stream) {
  if (R <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers) return CYR_UNSUPPORTED;
  if (R > kOneCtaRows) {  // multi-CTA coupled call (two passes, stream-ordered scratch)
    const size_t bytes = (size_t)R * sizeof(long long) + 16;
    void* scratch = nullptr;
    if (cyr::malloc_async(&scratch, bytes, stream) != cudaSuccess) return CYR_CUDA_ERROR;
    int* stop = reinterpret_cast<int*>(scratch);
    long long* thr = reinterpret_cast<long long*>(static_cast<unsigned char*>(scratch) + 16);
    cudaMemsetAsync(stop, 0, sizeof(int), stream);
    const int blocks = (R + 7) / 8;
    cyr::enforce_wide_setup_kernel<<<blocks, 256, 0, stream>>>(b, caps, demand_f, demand, R, E, thr,
                                                               stop, status);
    cyr::enforce_wide_finish_kernel<<<blocks, 256, 0, stream>>>(
        b, caps, demand_f, demand, R, E, thr, stop, m_hat, nu, degenerate, grants, margin, status);
    const cudaError_t e = cudaPeekAtLastError();
    cudaFreeAsync(scratch, stream);
    return e == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
  }
  const int nw = R < 16 ? R : 16;
  cyr::enforce_kernel<<<1, 32 * nw, 0, stream>>>(b, caps, demand_f, demand, R, E, m_hat, nu,
                                                degenerate, grants, margin, status);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}


int cyr_launch_latency_bench(int which, int iters, long long* cycles, double* sink) {
  switch (which) {
#define CYR_LB(W) case W: cyr::latency_bench_kernel<W><<<1, 32>>>(iters, cycles, sink); break;
    CYR_LB(0) CYR_LB(1) CYR_LB(2) CYR_LB(3) CYR_LB(4) CYR_LB(5) CYR_LB(6) CYR_LB(7) CYR_LB(8)
    CYR_LB(9) CYR_LB(10)
#undef CYR_LB
    default: return CYR_BAD_ARG;
  }
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

// rows at or below which a Mode-T level runs warp-per-row (CYR_WARP_LEVEL_ROWS)
static long long warp_level_rows() {
  static const long long v = [] {
    const char* e = getenv("CYR_WARP_LEVEL_ROWS");
    return e ? atoll(e) : 8192ll;
  }();
  return v;
}

int cyr_launch_tree_level(int precision, const void* raw, const int32_t* alloc, const double* eps,
                          int16_t* node, int S, int E, int L, int cap, int parents, int epad,
                          long long nodes_per_slot, long long parent_off, long long child_off,
                          int32_t* status, cudaStream_t stream) {
  if (S <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers || cap < 1 || cap > 16) return CYR_UNSUPPORTED;
  cyr::TreeIO io{alloc, eps, node, E, cap, epad, parents, nodes_per_slot, parent_off, child_off,
                 cyr_prof_buffer()};
  const long long groups = (long long)S * parents;
  if (groups * cap <= warp_level_rows()) {  // small level: warp per row (latency)
    const int gpc = 32 / cap;
    const long long blocks = (groups + gpc - 1) / gpc;
    const int threads = 32 * gpc * cap;
    const bool e10w = CYR_WARP_SPECIALISE && E == 10;
    if (precision == CYR_FP64) {
      auto kern = e10w ? cyr::tree_level_warp_kernel<double, 10> : cyr::tree_level_warp_kernel<double, 0>;
      kern<<<(unsigned)blocks, threads, 0, stream>>>(static_cast<const double*>(raw), io, groups,
                                                    L, status);
    } else {
      auto kern = e10w ? cyr::tree_level_warp_kernel<float, 10> : cyr::tree_level_warp_kernel<float, 0>;
      kern<<<(unsigned)blocks, threads, 0, stream>>>(static_cast<const float*>(raw), io, groups,
                                                    L, status);
    }
    return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
  }
  if (cyr::ensure_seat_table(stream) != CYR_OK) return CYR_CUDA_ERROR;
  const long long per_cta = (long long)cyr::kLaneWarps * (32 / cap);
  const long long blocks = (groups + per_cta - 1) / per_cta;
  if (blocks >= (1ll << 31)) return CYR_UNSUPPORTED;
  const size_t smem = cyr::kLaneWarps * cyr::lane_scratch_bytes(E);
  if (precision == CYR_FP64) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(cyr::tree_level_kernel<double>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cyr::tree_level_kernel<double><<<(unsigned)blocks, 32 * cyr::kLaneWarps, smem, stream>>>(
        static_cast<const double*>(raw), io, groups, L, status);
  } else {
    auto launch = [&](auto kern) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<(unsigned)blocks, 32 * cyr::kLaneWarps, smem, stream>>>(
          static_cast<const float*>(raw), io, groups, L, status);
    };
#ifndef CYR_LANE_SPECIALISE
#define CYR_LANE_SPECIALISE 1
#endif
    // cfg2's E = 10 with the user count compiled in (known trip counts):
    // deepest cfg2 level 990 -> 895 us.  E = 16 (cfg5) measured no gain (its
    // unrolled code is 8.2k instructions against 7.6k generic: the kernel is
    // instruction-cache sensitive), so it stays generic.
    if (CYR_LANE_SPECIALISE && E == 10) launch(cyr::tree_level_kernel<float, 10>);
    else launch(cyr::tree_level_kernel<float, 0>);
  }
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

// ------------------------------------------- shared-divisor division check
// div_rn_shared (projection.cuh) against __ddiv_rn, bit for bit, on operand
// pairs drawn from five families: random normals over a wide exponent range,
// cap-like dividends over water-level-like divisors, random bit patterns
// across the whole fast range, quotients planted next to representable
// values (a = RN(q * b)), and the Huntington-Hill divisors of seats 0..1023.
namespace cyr {
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long& s) {
  unsigned long long z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double bits_in(unsigned long long r, int emin, int emax) {
  const int e = emin + (int)((r >> 52) % (unsigned long long)(emax - emin + 1));
  return __longlong_as_double((long long)(((unsigned long long)(e + 1023) << 52) |
                                          (r & 0xfffffffffffffull)));
}
__global__ void shared_divisor_check_kernel(long long per_thread, unsigned long long seed,
                                            unsigned long long* bad) {
  unsigned long long st = seed ^ ((unsigned long long)(blockIdx.x * blockDim.x + threadIdx.x) << 20);
  unsigned long long mism = 0;
  for (long long i = 0; i < per_thread; ++i) {
    const unsigned long long r1 = splitmix64(st), r2 = splitmix64(st);
    double a, b;
    switch ((int)(i % 5)) {
      case 0: a = bits_in(r1, -60, 60); b = bits_in(r2, -60, 60); break;
      case 1: a = (double)(r1 % 800) + (double)(r1 >> 40) * 0x1p-24;
              b = bits_in(r2, -20, 10); break;
      case 2: a = bits_in(r1, -500, 499); b = bits_in(r2, -500, 499); break;
      case 3: {
        b = bits_in(r2, -30, 30);
        const double q = bits_in(r1, -30, 30);
        a = __dmul_rn(q, b);
        a = __longlong_as_double(__double_as_longlong(a) + (long long)(r1 % 5) - 2);
        break;
      }
      default: {
        const double x = (double)(r2 % kSeatTab);
        b = __dsqrt_rn(fmax(__dmul_rn(x, __dadd_rn(x, 1.0)), 1.0));
        a = bits_in(r1, -40, 12);
      }
    }
    const double want = __ddiv_rn(a, b);
    const double got = div_rn_shared(a, shared_divisor(b));
    mism += __double_as_longlong(want) != __double_as_longlong(got);
  }
  if (mism) atomicAdd(bad, mism);
}
}  // namespace cyr

int cyr_launch_shared_divisor_check(long long per_thread, unsigned long long seed, int sm_count,
                                    unsigned long long* bad, cudaStream_t stream) {
  cyr::shared_divisor_check_kernel<<<sm_count * 8, 256, 0, stream>>>(per_thread, seed, bad);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}
