// codebook.cu — K3: fused action -> codebook (and the standalone enforcer).
//
// Replaces, on the device and bit-exactly for identical float64 inputs:
//   neural.split_head / sample_squashed      neural.py:144-165
//   sac.policy_branch_actions head           sac.py:348-355
//   neural.action_to_scs                     neural.py:181-183
//   enforcer.kl_project_batch                enforcer.py:49-115
//   enforcer.apportion_batch                 enforcer.py:118-165
//
// Mapping: one warp per enforcement row, one lane per eMBB user (E <= 32).
// All rows of ONE coupled call live in one CTA: the bisection stop test of
// the reference is taken over every bisecting row of the call
// (enforcer.py:90-92), so converged rows keep bisecting until the last one
// converges; __syncthreads_or reproduces that exactly.
//
// Huntington-Hill: instead of materialising and lexsorting ~N seats per row
// (enforcer.py:147-164) each lane keeps its user's seat count; a warp
// argmax/argmin exchange moves the count vector to the exact top-`want` set
// of the reference order (phase, priority desc, user asc, seat asc).  Within
// a user the priorities m/sqrt(s(s+1)) strictly decrease, so the top set is a
// per-user prefix and the exchange converges to it; priorities are computed
// with the reference's exact float64 expression.
#include "cyrus_internal.cuh"
#include "cyrus_b200.h"

#include <math_constants.h>

namespace cyr {

struct Row {
  double b, c, d;  // this lane's raw action and cap; the row demand
  bool valid;      // row exists (warp-uniform)
  bool bis, degen; // warp-uniform
  double lo, hi;   // bisection bracket (identical in all lanes)
};

__device__ __forceinline__ bool lane_pos(const Row& r, int E) {
  return ((int)(threadIdx.x & 31) < E) && (r.b > kMassFloor) && (r.c > 0.0);
}

__device__ __forceinline__ void kl_setup(Row& r, int E) {
  const bool in = (int)(threadIdx.x & 31) < E;
  const bool pos = lane_pos(r, E);
  const double pos_cap = np_row_sum(pos ? r.c : 0.0, E);
  const bool active = r.valid && r.d > 0.0;
  r.degen = active && (pos_cap < __dsub_rn(r.d, 1e-12));
  r.bis = active && !r.degen;
  r.lo = 0.0;
  r.hi = 0.0;
  if (r.bis) {
    const double ratio = pos ? __ddiv_rn(r.b, fmax(r.c, 1e-300)) : CUDART_INF;
    const double lo = warp_min_d(in ? ratio : CUDART_INF);
    const double hi = __ddiv_rn(np_row_sum(in ? r.b : 0.0, E), r.d);
    r.lo = fmin(lo, hi);
    r.hi = hi;
  }
}

__device__ __forceinline__ bool kl_converged(const Row& r) {
  return !r.bis || (__dsub_rn(r.hi, r.lo) <= __dmul_rn(kRelWidth, r.hi));
}

__device__ __forceinline__ void kl_step(Row& r, int E) {
  if (!r.bis) return;
  const bool in = (int)(threadIdx.x & 31) < E;
  const double mid = __dmul_rn(__dsqrt_rn(r.lo), __dsqrt_rn(r.hi));
  const double q = in ? fmin(r.c, __ddiv_rn(r.b, mid)) : 0.0;
  const double fill = np_row_sum(q, E);
  if (fill >= r.d)
    r.lo = mid;
  else
    r.hi = mid;
}

// Coupled bisection of all rows held by the CTA; returns the iteration count.
template <int RPW>
__device__ int kl_group(Row (&rows)[RPW], int E) {
#pragma unroll
  for (int k = 0; k < RPW; ++k) kl_setup(rows[k], E);
  int it = 0;
  for (; it < kMaxIters; ++it) {
    bool conv = true;
#pragma unroll
    for (int k = 0; k < RPW; ++k) conv = conv && kl_converged(rows[k]);
    if (!__syncthreads_or(conv ? 0 : 1)) break;
#pragma unroll
    for (int k = 0; k < RPW; ++k) kl_step(rows[k], E);
  }
  return it;
}

// m_hat lane value and row nu after the bisection (enforcer.py:98-114).
__device__ __forceinline__ void kl_finish(const Row& r, int E, double& m, double& nu) {
  const bool in = (int)(threadIdx.x & 31) < E;
  m = 0.0;
  nu = 0.0;
  if (r.bis) {
    nu = __dmul_rn(__dsqrt_rn(r.lo), __dsqrt_rn(r.hi));
    m = in ? fmin(r.c, __ddiv_rn(r.b, nu)) : 0.0;
  } else if (r.degen) {
    const bool pos = lane_pos(r, E);
    double fill = pos ? r.c : 0.0;
    const double slack = __dsub_rn(r.d, np_row_sum(fill, E));
    const double spare = np_row_sum((in && !pos) ? r.c : 0.0, E);
    if (spare > 0.0 && slack > 0.0 && in && !pos) fill = __ddiv_rn(__dmul_rn(r.c, slack), spare);
    m = in ? fill : 0.0;
  }
}

// ------------------------------------------------------------ Huntington-Hill
__device__ __forceinline__ double seat_prio(double m, int seat) {
  const double a = (double)seat;
  return __ddiv_rn(m, __dsqrt_rn(fmax(__dmul_rn(a, __dadd_rn(a, 1.0)), 1.0)));
}

// (pa, la) strictly before (pb, lb) in the reference order within one phase.
__device__ __forceinline__ bool precedes(double pa, int la, double pb, int lb) {
  return pa > pb || (pa == pb && la < lb);
}

// first (best) candidate of the warp
__device__ __forceinline__ void warp_first(double& p, int& l, bool& ok) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double po = __shfl_xor_sync(kFull, p, off);
    const int lo = __shfl_xor_sync(kFull, l, off);
    const bool oko = __shfl_xor_sync(kFull, (int)ok, off);
    if (oko && (!ok || precedes(po, lo, p, l))) {
      p = po;
      l = lo;
      ok = true;
    }
  }
}

// last (worst) candidate of the warp
__device__ __forceinline__ void warp_last(double& p, int& l, bool& ok) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double po = __shfl_xor_sync(kFull, p, off);
    const int lo = __shfl_xor_sync(kFull, l, off);
    const bool oko = __shfl_xor_sync(kFull, (int)ok, off);
    if (oko && (!ok || precedes(p, l, po, lo))) {
      p = po;
      l = lo;
      ok = true;
    }
  }
}

// Seats granted to this lane's user; `margin` gets the relative priority gap
// between the last granted and first refused seat of the same positive phase
// (+inf otherwise) — the near-tie score of SURVEY §8(c).
__device__ int hh_row(double m, double c, int E, long long want, double& margin) {
  const int lane = threadIdx.x & 31;
  const bool in = lane < E;
  const int cnt = in ? (int)ceil(c) : 0;
  const bool posu = in && m > 0.0 && cnt >= 1;
  margin = CUDART_INF;
  if (want <= 0) return 0;
  const unsigned posmask = __ballot_sync(kFull, posu);
  const int n0 = __popc(posmask);

  if (want <= n0) {  // phase 0 only: first seats by mass
    int rank = 0;
    for (int f = 0; f < 32; ++f) {
      const double mf = shfl_d(m, f);
      if (((posmask >> f) & 1u) && precedes(mf, f, m, lane)) ++rank;
    }
    const unsigned lastm = __ballot_sync(kFull, posu && rank == want - 1);
    const unsigned nextm = __ballot_sync(kFull, posu && rank == want);
    const double m_last = shfl_d(m, lastm ? __ffs(lastm) - 1 : 0);
    const double m_next = shfl_d(m, nextm ? __ffs(nextm) - 1 : 0);
    if (nextm && lastm) margin = __ddiv_rn(__dsub_rn(m_last, m_next), m_last);
    return (posu && rank < want) ? 1 : 0;
  }

  const int r1 = (int)(want - n0);
  const int p1 = __reduce_add_sync(kFull, posu ? cnt - 1 : 0);
  if (r1 <= p1) {  // exact top-r1 of phase 1 by exchange
    int h = 0;
    if (posu) {
      int g = (int)floor(m);
      if (g >= 1 && (double)g * (double)(g + 1) > m * m) g -= 1;
      h = max(0, min(g, cnt - 1));
    }
    const int guard = 256 + 4 * r1;
    for (int step = 0; step < guard; ++step) {
      const int total = __reduce_add_sync(kFull, h);
      bool oka = posu && (h + 1 <= cnt - 1);
      double pa = oka ? seat_prio(m, h + 1) : 0.0;
      int la = lane;
      bool okd = posu && h >= 1;
      double pd = okd ? seat_prio(m, h) : 0.0;
      int ld = lane;
      warp_first(pa, la, oka);
      warp_last(pd, ld, okd);
      if (total < r1) {
        if (lane == la) ++h;
      } else if (total > r1) {
        if (lane == ld) --h;
      } else if (oka && okd && precedes(pa, la, pd, ld)) {
        if (lane == la) ++h;
        if (lane == ld) --h;
      } else {
        if (oka && okd) margin = __ddiv_rn(__dsub_rn(pd, pa), pd);
        break;
      }
    }
    return posu ? 1 + h : 0;
  }

  // every positive-mass user is full; zero-mass users take first seats in
  // index order (phase 2), then all later seats user by user (phase 3)
  int g = posu ? cnt : 0;
  const bool zu = in && !(m > 0.0) && cnt >= 1;
  const unsigned zmask = __ballot_sync(kFull, zu);
  const int r2 = r1 - p1;
  const int rank2 = __popc(zmask & ((1u << lane) - 1u));
  if (zu && rank2 < r2) g += 1;
  const int r3 = r2 - __popc(zmask);
  if (r3 > 0) {
    const int extra = zu ? cnt - 1 : 0;
    int incl = extra;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, off);
      if (lane >= off) incl += y;
    }
    const int before = incl - extra;
    if (zu) g += max(0, min(extra, r3 - before));
  }
  return g;
}

__device__ __forceinline__ void set_status(int32_t* status, int code) {
  if (status) atomicMax(status, code);
}

// ------------------------------------------------------------ codebook K3
template <typename RawT>
__global__ void __launch_bounds__(1024) codebook_kernel(
    const RawT* __restrict__ raw, const int32_t* __restrict__ alloc,
    const double* __restrict__ eps, int E, int L, int cap, int32_t* __restrict__ cb,
    double* __restrict__ m_out, double* __restrict__ nu_out, double* __restrict__ margin_out,
    int32_t* __restrict__ iters_out, int32_t* __restrict__ status) {
  const int s = blockIdx.x;
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool in = lane < E;
  const long long col = (long long)s * cap + w;

  const double n = in ? (double)alloc[(long long)s * E + lane] : 0.0;
  double bval = 0.0;
  if (in) {
    const double mu = (double)raw[col * 2 * E + lane];
    const double ls = fmin(fmax((double)raw[col * 2 * E + E + lane], kLogSigmaMin), kLogSigmaMax);
    double a;
    if (eps != nullptr) {
      const double u = __dadd_rn(mu, __dmul_rn(exp(ls), eps[col * E + lane]));
      a = tanh(u);
    } else {
      a = tanh(mu);
    }
    bval = __dmul_rn(__dmul_rn(__dadd_rn(a, 1.0), 0.5), n);
  }
  Row rows[1];
  rows[0].b = bval;
  rows[0].c = n;
  rows[0].d = (double)((long long)(w + 1) * L);
  rows[0].valid = true;
  const double capsum = np_row_sum(n, E);  // enforcer.py:64 / :138
  if (lane == 0 && rows[0].d > capsum) set_status(status, CYR_INFEASIBLE);

  const int iters = kl_group<1>(rows, E);
  double m, nu;
  kl_finish(rows[0], E, m, nu);
  double margin;
  const int g = hh_row(m, n, E, (long long)(w + 1) * L, margin);

  int32_t* book = cb + (long long)s * (cap + 1) * E;
  if (in) {
    book[(long long)(w + 1) * E + lane] = g;
    if (w == 0) book[lane] = 0;
    if (m_out) m_out[col * E + lane] = m;
  }
  if (lane == 0) {
    if (nu_out) nu_out[col] = nu;
    if (margin_out) margin_out[col] = margin;
    if (iters_out && w == 0) iters_out[s] = iters;
  }
}

// ------------------------------------------------------- standalone enforcer
template <int RPW>
__global__ void __launch_bounds__(1024) enforce_kernel(
    const double* __restrict__ b, const double* __restrict__ caps,
    const double* __restrict__ demand_f, const int64_t* __restrict__ demand, int R, int E,
    double* __restrict__ m_out,
    double* __restrict__ nu_out, uint8_t* __restrict__ degen_out, int64_t* __restrict__ grants,
    double* __restrict__ margin_out, int32_t* __restrict__ status) {
  const int nw = blockDim.x >> 5;
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool in = lane < E;
  Row rows[RPW];
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int r = w + k * nw;
    Row& row = rows[k];
    row.valid = r < R;
    row.b = (row.valid && in) ? b[(long long)r * E + lane] : 0.0;
    row.c = (row.valid && in) ? caps[(long long)r * E + lane] : 0.0;
    row.d = row.valid ? (demand_f ? demand_f[r] : (double)demand[r]) : 0.0;
    if (row.valid) {
      const bool neg = __any_sync(kFull, row.b < 0.0 || row.c < 0.0) || row.d < 0.0;
      const double capsum = np_row_sum(row.c, E);
      if (lane == 0) {
        if (neg) set_status(status, CYR_BAD_ARG);
        else if (demand_f ? row.d > __dadd_rn(capsum, 1e-9) : row.d > capsum)
          set_status(status, CYR_INFEASIBLE);  // enforcer.py:64 / :138
      }
    }
  }
  kl_group<RPW>(rows, E);
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int r = w + k * nw;
    if (!rows[k].valid) continue;  // warp-uniform
    double m, nu;
    kl_finish(rows[k], E, m, nu);
    double margin = CUDART_INF;
    int g = 0;
    if (grants) g = hh_row(m, rows[k].c, E, demand[r], margin);  // warp-uniform
    if (in) {
      if (m_out) m_out[(long long)r * E + lane] = m;
      if (grants) grants[(long long)r * E + lane] = g;
    }
    if (lane == 0) {
      if (nu_out) nu_out[r] = nu;
      if (degen_out) degen_out[r] = rows[k].degen ? 1 : 0;
      if (margin_out) margin_out[r] = margin;
    }
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

}  // namespace cyr

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
  if (E < 1 || E > cyr::kMaxUsers || cap < 1 || cap > 32) return CYR_UNSUPPORTED;
  const dim3 grid(S), block(32 * cap);
  if (precision == CYR_FP64)
    cyr::codebook_kernel<double><<<grid, block, 0, stream>>>(
        static_cast<const double*>(raw), alloc, eps, E, L, cap, codebook, m_hat, nu, margin, iters,
        status);
  else
    cyr::codebook_kernel<float><<<grid, block, 0, stream>>>(
        static_cast<const float*>(raw), alloc, eps, E, L, cap, codebook, m_hat, nu, margin, iters,
        status);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

int cyr_launch_enforce(const double* b, const double* caps, const double* demand_f,
                       const int64_t* demand, int R, int E,
                       double* m_hat, double* nu, uint8_t* degenerate, int64_t* grants,
                       double* margin, int32_t* status, cudaStream_t stream) {
  if (R <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers || R > 256) return CYR_UNSUPPORTED;
  const int nw = R < 32 ? R : 32;
  const int rpw = (R + nw - 1) / nw;
  const dim3 block(32 * nw);
#define CYR_ENFORCE(K)                                                                        \
  cyr::enforce_kernel<K><<<1, block, 0, stream>>>(b, caps, demand_f, demand, R, E, m_hat, nu, degenerate, \
                                                   grants, margin, status)
  if (rpw <= 1) CYR_ENFORCE(1);
  else if (rpw <= 2) CYR_ENFORCE(2);
  else if (rpw <= 4) CYR_ENFORCE(4);
  else CYR_ENFORCE(8);
#undef CYR_ENFORCE
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}
