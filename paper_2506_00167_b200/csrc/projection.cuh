// projection.cuh — K3 device code shared by the batch codebook kernel, the
// standalone enforcer kernels and the fused single-slot latency kernel.
//
// Replaces, on the device and bit-exactly for identical float64 inputs:
//   neural.split_head / sample_squashed      neural.py:144-165
//   sac.policy_branch_actions head           sac.py:348-355
//   neural.action_to_scs                     neural.py:181-183
//   enforcer.kl_project_batch                enforcer.py:49-115
//   enforcer.apportion_batch                 enforcer.py:118-165
//
// Mapping: one warp per enforcement row, one lane per eMBB user (E <= 32),
// for the per-row phases; the coupled bisection of a call runs with one lane
// per row (see coupled_bisection / codebook_rows).
//
// Huntington-Hill: instead of materialising and lexsorting ~N seats per row
// (enforcer.py:147-164) each lane keeps its user's seat count; a warp
// argmax/argmin exchange moves the count vector to the exact top-`want` set
// of the reference order (phase, priority desc, user asc, seat asc).  Within
// a user the priorities m/sqrt(s(s+1)) strictly decrease, so the top set is a
// per-user prefix and the exchange converges to it; priorities are computed
// with the reference's exact float64 expression.
#pragma once

#include "cyrus_internal.cuh"
#include "cyrus_b200.h"

#include <math_constants.h>

namespace cyr {

// a / b for b positive, normal and finite.  A zero dividend (padding lanes,
// zero-mass users) would send __ddiv_rn down its slow path and stall the
// whole warp; 0 / b is exactly +0, so such lanes divide a dummy and select 0.
__device__ __forceinline__ double div_or_zero(double a, double b) {
  const double q = __ddiv_rn(a != 0.0 ? a : 1.0, b);
  return a != 0.0 ? q : 0.0;
}

// Division by a divisor shared by many dividends (one fill evaluation divides
// a row's E masses by one water level; the Huntington-Hill priorities divide
// by per-seat constants): y = RN(1/b) once (__drcp_rn), then per dividend
// q0 = RN(a*y), one Newton correction q1 = RN(q0 + (a - b*q0)*y), and
// Markstein's final step q = RN(q1 + (a - b*q1)*y) -- the remainders exact by
// FMA.  With y within half an ulp of 1/b and q1 within one ulp of a/b, that
// step returns RN(a/b) (Markstein 1990; Muller et al., Handbook of
// Floating-Point Arithmetic, "Markstein's theorem"), i.e. the bits of
// __ddiv_rn.  The operands are held to [2^-500, 2^500] so no quotient,
// product or remainder leaves the normal range; anything else (zero,
// subnormal, huge, inf, NaN) takes __ddiv_rn.  cyr_selftest_shared_divisor
// compares the two on 2^30+ operand pairs (tests/test_gpu_guards.py).
struct SharedDivisor {
  double b, y;
  bool fast;
};
__device__ __forceinline__ bool markstein_range(double v) {
  return v >= 0x1p-500 && v <= 0x1p500;
}
__device__ __forceinline__ SharedDivisor shared_divisor(double b) {
  SharedDivisor s;
  s.b = b;
  s.fast = markstein_range(b);
  s.y = s.fast ? __drcp_rn(b) : 0.0;
  return s;
}
__device__ __forceinline__ SharedDivisor shared_divisor(double b, double y) {  // y = __drcp_rn(b)
  SharedDivisor s;
  s.b = b;
  s.y = y;
  s.fast = markstein_range(b);
  return s;
}
__device__ __forceinline__ double div_rn_shared(double a, const SharedDivisor& s) {
  if (s.fast && markstein_range(a)) {
    double q = __dmul_rn(a, s.y);
    q = __fma_rn(__fma_rn(-q, s.b, a), s.y, q);
    return __fma_rn(__fma_rn(-q, s.b, a), s.y, q);
  }
  return __ddiv_rn(a, s.b);
}
// div_or_zero(a, s.b), bit for bit
__device__ __forceinline__ double div_or_zero(double a, const SharedDivisor& s) {
  return a != 0.0 ? div_rn_shared(a, s) : 0.0;
}

struct Row {
  double b, c, d;  // this lane's raw action and cap; the row demand
  bool valid;      // row exists (warp-uniform)
  bool bis, degen; // warp-uniform
  bool full;       // bisecting with demand >= every usable cap: all users end capped
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
  r.full = r.bis && pos_cap <= r.d;
  r.lo = 0.0;
  r.hi = 0.0;
  if (r.bis) {
    const double ratio = pos ? __ddiv_rn(pos ? r.b : 1.0, pos ? fmax(r.c, 1e-300) : 1.0)
                             : CUDART_INF;
    const double lo = warp_min_d(in ? ratio : CUDART_INF);
    const double hi = __ddiv_rn(np_row_sum(in ? r.b : 0.0, E), r.d);
    r.lo = fmin(lo, hi);
    r.hi = hi;
  }
}

// ----------------------------------------------------------- exact bisection
// The reference bisects (enforcer.py:90-97): mid = sqrt(lo)*sqrt(hi),
// fill = rowsum(min(c, b/mid)), lo = mid if fill >= d else hi = mid.  The
// computed predicate P(x) = [rowsum(min(c, b/x)) >= d] is EXACTLY monotone
// in x: IEEE division is correctly rounded hence monotone in the divisor,
// min(c, .) is monotone, and fixed-order float additions of non-negative
// terms are monotone in every term.  So there is one threshold bit pattern
// T per row with P(x) <=> bits(x) <= T (positive doubles order like their
// bit patterns), and every bisection decision of the reference equals the
// integer compare bits(mid) <= T.  T is found with a few exact evaluations
// of P around the analytic water level; the 40-50 coupled bisection steps
// then cost one sqrt and one multiply each instead of an fp64 division, a
// shuffle-tree row sum and a CTA barrier.

// P(x), evaluated with the reference's exact float64 expression.
__device__ __forceinline__ bool fill_reaches(const Row& r, int E, double x) {
  const bool in = (int)(threadIdx.x & 31) < E;
  const double q = in ? fmin(r.c, div_or_zero(r.b, x)) : 0.0;
  return np_row_sum(q, E) >= r.d;
}

__device__ __forceinline__ double warp_sum_d(double v) {  // any order: estimate only
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  return v;
}

// Water level of the exact-arithmetic projection: fixed point of
// nu = sum_uncapped(b) / (d - sum_capped(c)), capped <=> b >= nu*c.
static __device__ double water_level(const Row& r, int E) {
  // demand = every usable cap (the j = cap row when N = cap * L): the level
  // sits at the smallest cap ratio, lo; the fixed point below would take
  // one iteration per user to get there
  if (r.full) return r.lo;
  const bool in = (int)(threadIdx.x & 31) < E;
  const bool pos = lane_pos(r, E);
  double nu = r.hi;
  unsigned prev = 0xffffffffu;
  for (int it = 0; it <= E; ++it) {
    const bool capped = pos && (r.b >= nu * r.c);
    const unsigned mask = __ballot_sync(kFull, capped);
    if (mask == prev) break;
    prev = mask;
    const double cc = warp_sum_d(capped ? r.c : 0.0);
    const double bu = warp_sum_d((in && !capped) ? r.b : 0.0);
    const double den = r.d - cc;
    if (den <= 0.0) {  // everything left is capped: the level sits at a cap ratio
      nu = warp_min_d(capped ? (capped ? r.b : 1.0) / (capped ? fmax(r.c, 1e-300) : 1.0)
                             : CUDART_INF);
      break;
    }
    nu = bu / den;
  }
  if (!(nu > 0.0) || isinf(nu)) nu = sqrt(r.lo) * sqrt(r.hi);
  return nu;
}

// Largest positive-double bit pattern T with P(from_bits(T)) true, found by
// galloping from x0 then halving on the integer bit patterns.  P(+0) is
// true (fill = sum of usable caps >= d for a bisecting row) and P(+inf) is
// false (fill = 0 < d), so the search is always bracketed.
static __device__ long long fill_threshold(const Row& r, int E, double x0) {
  constexpr long long kInf = 0x7ff0000000000000ll;
  long long lo, hi;  // P(lo) true, P(hi) false
  const long long a = __double_as_longlong(x0);
  if (fill_reaches(r, E, x0)) {
    lo = a;
    for (long long step = 1;; step <<= 1) {
      const long long cand = lo + step;
      if (cand >= kInf) { hi = kInf; break; }
      if (!fill_reaches(r, E, __longlong_as_double(cand))) { hi = cand; break; }
      lo = cand;
    }
  } else {
    hi = a;
    for (long long step = 1;; step <<= 1) {
      const long long cand = hi - step;
      if (cand <= 0) { lo = 0; break; }
      if (fill_reaches(r, E, __longlong_as_double(cand))) { lo = cand; break; }
      hi = cand;
    }
  }
  while (hi - lo > 1) {
    const long long mid = lo + ((hi - lo) >> 1);
    if (fill_reaches(r, E, __longlong_as_double(mid))) lo = mid;
    else hi = mid;
  }
  return lo;
}

// The reference's coupled loop with lanes = rows (RPL rows per lane): a
// call stops when every bisecting row satisfies hi - lo <= 1e-13*hi
// (enforcer.py:91).  `group` > 0 splits the warp's rows into independent
// calls of `group` consecutive lanes (one slot each, RPL == 1); group == 0
// couples every row.  Returns the iteration count of this lane's call.
template <int RPL, bool SKIP = false>
__device__ int coupled_bisection(double (&lo)[RPL], double (&hi)[RPL], const long long (&T)[RPL],
                                 const bool (&bis)[RPL], int group = 0) {
  // Chunks of kSpec steps run speculatively with the bracket history kept in
  // registers; the stop test (one vote per chunk instead of per step) then
  // picks the exact iteration where the reference loop would have stopped
  // and rolls the bracket back to it.  The serial chain per step is one
  // DMUL and one correctly rounded sqrt.
#ifndef CYR_SPEC
#define CYR_SPEC 4  // steps per speculative chunk (2 / 4 / 6 / 8 / 16 A/B: 4 best by ~1 us on the batch K3)
#endif
  constexpr int kSpec = RPL == 1 ? CYR_SPEC : 1;
  const int lane = threadIdx.x & 31;
  double sl[RPL], sh[RPL];
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    sl[k] = bis[k] ? __dsqrt_rn(lo[k]) : 0.0;
    sh[k] = bis[k] ? __dsqrt_rn(hi[k]) : 0.0;
  }
  const unsigned gmask =
      group > 0 ? (((group >= 32) ? kFull : ((1u << group) - 1u)) << (lane - lane % group)) : kFull;
  auto converged = [&](const double (&l)[RPL], const double (&h)[RPL]) {
    bool conv = true;
#pragma unroll
    for (int k = 0; k < RPL; ++k)
      conv = conv && (!bis[k] || __dsub_rn(h[k], l[k]) <= __dmul_rn(kRelWidth, h[k]));
    return conv;
  };
  // SKIP (the lane-mapped K3 of big batches and Mode-T levels, where it saves
  // 3-4 % of the tree; on the warp-per-row paths the plain step loop measured
  // slower than the speculative chunks): steps that provably precede the stop
  // run without history or votes.  The
  // bracket is a bisection in log space: ln(hi/lo) halves per step up to the
  // rounding of one sqrt and one multiply (a relative deviation of ~1.5 ulp
  // against a width >= 450 ulp while not converged), and the stop test needs
  // ln(hi/lo) <~ 1e-13.  So a row cannot converge before
  // floor(log2(ln(hi0/lo0) / 1e-13)) steps; 3 steps of margin absorb the
  // rounding.  The warp skips the minimum of that bound over its bisecting
  // lanes; every step it skips is computed exactly as below, so the results
  // and the stop iteration are unchanged.
  // (cheap bounds from the exponent and mantissa bits: with x = 2^e (1 + f),
  // e + f <= log2 x <= e + f / ln 2)
  auto split = [](double x, double& f) {
    const long long b = __double_as_longlong(x);
    f = __longlong_as_double((b & 0xfffffffffffffll) | 0x3ff0000000000000ll) - 1.0;
    return (int)((b >> 52) & 0x7ff) - 1023;
  };
  int tl = kMaxIters;
  bool anyb = false;
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    if (!bis[k]) continue;
    anyb = true;
    int t = 0;
    if (lo[k] > 2.3e-308 && hi[k] < 1e308) {  // normal numbers
      double fh, fl;
      const int eh = split(hi[k], fh), el = split(lo[k], fl);
      // lower bound of ln(hi/lo)
      const double lr = 0.6931471805599453 * ((double)(eh - el) + fh - fl * 1.4426950408889634);
      if (lr > 0.0) {
        double fy;
        t = split(lr * 1e13, fy) - 3;  // floor(log2(lr / 1e-13)) - 3
      }
    }
    tl = min(tl, max(t, 0));
  }
  int tskip = __reduce_min_sync(kFull, anyb ? tl : kMaxIters);
  if (tskip >= kMaxIters || !SKIP) tskip = 0;  // no lane bisects / not enabled
#pragma unroll 8
  for (int t = 0; t < tskip; ++t) {
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const double mid = __dmul_rn(sl[k], sh[k]);
      const double root = __dsqrt_rn(mid);
      const bool up = bis[k] && __double_as_longlong(mid) <= T[k];
      const bool dn = bis[k] && !up;
      lo[k] = up ? mid : lo[k];
      sl[k] = up ? root : sl[k];
      hi[k] = dn ? mid : hi[k];
      sh[k] = dn ? root : sh[k];
    }
  }
  // a call without bisecting rows stops at 0 (its brackets never move)
  const bool group_bis = (__ballot_sync(kFull, anyb) & gmask) != 0u;

  bool frozen = false;
  int stop = kMaxIters;
  for (int base = tskip; base < kMaxIters; base += kSpec) {
    double hl[kSpec + 1][RPL], hh[kSpec + 1][RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      hl[0][k] = lo[k];
      hh[0][k] = hi[k];
    }
    if (!frozen) {
#pragma unroll
      for (int t = 0; t < kSpec; ++t) {
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const double mid = __dmul_rn(sl[k], sh[k]);
          const double root = __dsqrt_rn(mid);  // needed on either side: no divergence
          const bool up = bis[k] && __double_as_longlong(mid) <= T[k];
          const bool dn = bis[k] && !up;
          lo[k] = up ? mid : lo[k];
          sl[k] = up ? root : sl[k];
          hi[k] = dn ? mid : hi[k];
          sh[k] = dn ? root : sh[k];
          hl[t + 1][k] = lo[k];
          hh[t + 1][k] = hi[k];
        }
      }
    }
    // first state t of this chunk at which this lane's call has converged
    // (one ballot per state; a segmented shuffle AND of per-lane bitmasks and
    // a REDUX-max of first-converged states both measured slower: 8.0 and
    // 10.6 us vs 5.0 us for a 46-step call)
    int first = kSpec + 1;
#pragma unroll
    for (int t = kSpec; t >= 0; --t) {
      const unsigned done = __ballot_sync(kFull, frozen || converged(hl[t], hh[t]));
      if ((done & gmask) == gmask && base + t <= kMaxIters) first = t;
    }
    if (!frozen && first <= kSpec) {
      frozen = true;
      stop = base + first;
#pragma unroll
      for (int t = 0; t <= kSpec; ++t)
        if (t == first)
#pragma unroll
          for (int k = 0; k < RPL; ++k) {
            lo[k] = hl[t][k];
            hi[k] = hh[t][k];
          }
    }
    if (__all_sync(kFull, frozen)) break;
  }
  return group_bis ? stop : 0;
}

// m_hat lane value and row nu after the bisection (enforcer.py:98-114).
__device__ __forceinline__ void kl_finish(const Row& r, int E, double& m, double& nu) {
  const bool in = (int)(threadIdx.x & 31) < E;
  m = 0.0;
  nu = 0.0;
  if (r.bis) {
    nu = __dmul_rn(__dsqrt_rn(r.lo), __dsqrt_rn(r.hi));
    m = in ? fmin(r.c, div_or_zero(r.b, nu)) : 0.0;
  } else if (r.degen) {
    const bool pos = lane_pos(r, E);
    double fill = pos ? r.c : 0.0;
    const double slack = __dsub_rn(r.d, np_row_sum(fill, E));
    const double spare = np_row_sum((in && !pos) ? r.c : 0.0, E);
    if (spare > 0.0 && slack > 0.0 && in && !pos) fill = div_or_zero(__dmul_rn(r.c, slack), spare);
    m = in ? fill : 0.0;
  }
}

// ------------------------------------------------------------ Huntington-Hill
__device__ __forceinline__ double seat_prio(double m, int seat) {
  const double a = (double)seat;
  return div_or_zero(m, __dsqrt_rn(fmax(__dmul_rn(a, __dadd_rn(a, 1.0)), 1.0)));
}

// (pa, la) strictly before (pb, lb) in the reference order within one phase.
__device__ __forceinline__ bool precedes(double pa, int la, double pb, int lb) {
  return pa > pb || (pa == pb && la < lb);
}

// First (best) add candidate and last (worst) held seat of the warp, in one
// butterfly: (pa, la, oka) -> best, (pd, ld, okd) -> worst.
__device__ __forceinline__ void warp_first_last(double& pa, int& la, bool& oka, double& pd, int& ld,
                                                bool& okd) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double pao = __shfl_xor_sync(kFull, pa, off);
    const double pdo = __shfl_xor_sync(kFull, pd, off);
    const int packed = (la << 8) | (ld << 1);
    const int po = __shfl_xor_sync(kFull, packed | (oka ? 1 << 16 : 0) | (okd ? 1 : 0), off);
    const int lao = (po >> 8) & 0xff, ldo = (po >> 1) & 0x7f;
    const bool okao = (po >> 16) & 1, okdo = po & 1;
    if (okao && (!oka || precedes(pao, lao, pa, la))) {
      pa = pao;
      la = lao;
      oka = true;
    }
    if (okdo && (!okd || precedes(pd, ld, pdo, ldo))) {
      pd = pdo;
      ld = ldo;
      okd = true;
    }
  }
}

// Seats granted to this lane's user; `margin` gets the relative priority gap
// between the last granted and first refused seat of the same positive phase
// (+inf otherwise) — the near-tie score of SURVEY §8(c).
static __device__ int hh_row(double m, double c, int E, long long want, double& margin,
                             int* steps_out = nullptr) {
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
    if (nextm && lastm) margin = div_or_zero(__dsub_rn(m_last, m_next), m_last);
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
      warp_first_last(pa, la, oka, pd, ld, okd);
      if (total < r1) {
        if (lane == la) ++h;
      } else if (total > r1) {
        if (lane == ld) --h;
      } else if (oka && okd && precedes(pa, la, pd, ld)) {
        if (lane == la) ++h;
        if (lane == ld) --h;
      } else {
        if (oka && okd) margin = div_or_zero(__dsub_rn(pd, pa), pd);
        if (steps_out) *steps_out = step + 1;
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

// Any failing row stores its nonzero code (plain store: the buffer may be
// mapped host memory, and any nonzero code is a failure of the call).
__device__ __forceinline__ void set_status(int32_t* status, int code) {
  if (status) *reinterpret_cast<volatile int32_t*>(status) = code;
}

// ------------------------------------------------------- slot codebooks
// Head + coupled projection + rounding for `nrows` rows held by this CTA
// (warp w < nrows owns local row w = global row row0 + w).  Rows come in
// whole groups of `cap` (branch j = row % cap + 1, demand j*L) and each
// group is one coupled enforcement call: a slot's branch rows in Mode R
// (engine.py:108-110), a parent node's branch rows in Mode T.  Every thread
// of the CTA must call this (it uses __syncthreads); blockDim.x >= 32 *
// nrows, nrows <= 32, row0 % cap == 0.  raw points at local row 0's logits
// ([row][2E]).  IO supplies the group's allocation row and the row's noise
// and consumes the grants (lanes < E) — see SlotIO / the Mode-T TreeIO.
// Shared-memory scratch of one codebook_rows_io call (<= 32 rows).
struct RowScratch {
  double lo[32], hi[32];
  long long t[32];
  int flags[32];      // bit 0 bis, bit 1 degen
  int iters[32];
  double b[32][32];   // [row][user] raw actions from phase 1 (head computed once)
};

// Phase 1 of one row (whole warp, lane = user): head, bracket, water level,
// exact fill threshold.  Returns b (this lane's raw action); lo/hi/threshold
// and flags go to the caller's scratch through the out-parameters.
template <typename RawT, typename IO>
__device__ __forceinline__ double row_phase1(const RawT* rr, long long grow, int cap, int E, int L,
                                             const IO& io, int32_t* status, double& lo_out,
                                             double& hi_out, long long& thr_out, int& flags_out,
                                             unsigned long long* tr = nullptr) {
  const int lane = threadIdx.x & 31;
  const bool in = lane < E;
  const long long group = grow / cap;
  const int j = (int)(grow % cap) + 1;
  const int32_t* alloc = io.alloc_row(group);
  const double* eps = io.eps_row(grow, group, j);
  Row row;
  row.valid = true;
  const double n = in ? (double)alloc[lane] : 0.0;
  double bval = 0.0;
  if (in) {
    const double mu = (double)rr[lane];
    const double ls = fmin(fmax((double)rr[E + lane], kLogSigmaMin), kLogSigmaMax);
    double a;
    if (eps != nullptr) {
      const double u = __dadd_rn(mu, __dmul_rn(exp(ls), eps[lane]));
      a = tanh(u);
    } else {
      a = tanh(mu);
    }
    bval = __dmul_rn(__dmul_rn(__dadd_rn(a, 1.0), 0.5), n);  // neural.py:181-183
  }
  row.b = bval;
  row.c = n;
  row.d = (double)((long long)j * L);
  const double capsum = np_row_sum(n, E);  // enforcer.py:64 / :138
  if (lane == 0 && row.d > capsum) set_status(status, CYR_INFEASIBLE);
  trace_stamp(tr, 8);
  kl_setup(row, E);
  trace_stamp(tr, 9);
  long long thr = 0;
  if (row.bis) thr = fill_threshold(row, E, water_level(row, E));
  trace_stamp(tr, 10);
  lo_out = row.lo;
  hi_out = row.hi;
  thr_out = thr;
  flags_out = (row.bis ? 1 : 0) | (row.degen ? 2 : 0);
  return bval;
}

// Phase 3 of one row (whole warp): m_hat, nu, Huntington-Hill, emit.
template <typename IO>
__device__ __forceinline__ void row_phase3(long long grow, int cap, int E, int L, const IO& io,
                                           double bval, double lo, double hi, int flags, int iters,
                                           int lr = 0, unsigned long long* tr = nullptr) {
  const int lane = threadIdx.x & 31;
  const bool in = lane < E;
  const long long group = grow / cap;
  const int j = (int)(grow % cap) + 1;
  const int32_t* alloc = io.alloc_row(group);
  Row row;
  row.valid = true;
  row.b = bval;
  row.c = in ? (double)alloc[lane] : 0.0;
  row.d = (double)((long long)j * L);
  row.bis = (flags & 1) != 0;
  row.degen = (flags & 2) != 0;
  row.lo = lo;
  row.hi = hi;
  double m, nu;
  kl_finish(row, E, m, nu);
  trace_stamp(tr, 13);
  double margin;
  int hh_steps = 0;
  const int g = hh_row(m, row.c, E, (long long)j * L, margin, &hh_steps);
  trace_stamp(tr, 14);
  if (lr < 8) trace_value(tr, 40 + lr, hh_steps);
  if (lr < 8) trace_value(tr, 56 + lr, iters);
  io.emit(grow, group, j, lane, g, m, nu, margin, iters);
}

// KE > 0: the user count compiled in (the warp row sums then shuffle only
// the lanes that exist: 6 instead of 14 shuffles per sum at E = 10)
template <typename RawT, typename IO, int KE = 0>
__device__ void codebook_rows_io(const RawT* raw, long long row0, int nrows, int cap, int E_rt,
                                 int L, const IO& io, int32_t* status, RowScratch& sc,
                                 unsigned long long* tr = nullptr) {
  const int E = KE > 0 ? KE : E_rt;
  const int w = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  // phase 1 (warp per row, warps stride over the rows)
  for (int lr = w; lr < nrows; lr += nw) {
    double lo, hi;
    long long thr;
    int flags;
    const double bval = row_phase1(raw + (long long)lr * 2 * E, row0 + lr, cap, E, L, io, status,
                                   lo, hi, thr, flags, tr);
    sc.b[lr][lane] = bval;
    if (lane == 0) {
      sc.lo[lr] = lo;
      sc.hi[lr] = hi;
      sc.t[lr] = thr;
      sc.flags[lr] = flags;
    }
    if (lr < 8) trace_stamp_warp(tr, 16 + lr);
  }
  __syncthreads();
  // phase 2 (warp 0, lanes = rows): the coupled loop of every group at once
  if (w == 0) {
    double lo[1] = {lane < nrows ? sc.lo[lane] : 0.0};
    double hi[1] = {lane < nrows ? sc.hi[lane] : 0.0};
    const long long tt[1] = {lane < nrows ? sc.t[lane] : 0};
    const bool bis[1] = {lane < nrows && (sc.flags[lane] & 1)};
    trace_stamp(tr, 11);
    const int iters = coupled_bisection<1>(lo, hi, tt, bis, cap);  // rows are group-aligned
    trace_stamp(tr, 12);
    if (lane < nrows) {
      sc.lo[lane] = lo[0];
      sc.hi[lane] = hi[0];
      sc.iters[lane] = iters;
    }
  }
  __syncthreads();
  // phase 3 (warp per row)
  for (int lr = w; lr < nrows; lr += nw)
    row_phase3(row0 + lr, cap, E, L, io, sc.b[lr][lane], sc.lo[lr], sc.hi[lr], sc.flags[lr],
               sc.iters[lr], lr, tr);
}

// One warp = one whole coupled call of `cap` rows (group `group`, rows
// group*cap ..): phase 1 row by row, the coupled loop with lanes = rows,
// phase 3 row by row — no CTA barrier, so the warps of a CTA (different
// groups) overlap their latency chains.  Scratch: this warp's slice.
struct WarpScratch {
  double lo[32], hi[32];
  long long t[32];
  int flags[32];
  int iters;
};

template <typename RawT, typename IO>
__device__ void codebook_group_warp(const RawT* raw, long long group, int cap, int E, int L,
                                    const IO& io, int32_t* status, WarpScratch& sc,
                                    double* bsc /* [cap][32] */) {
  const int lane = threadIdx.x & 31;
  const long long row0 = group * cap;
  for (int r = 0; r < cap; ++r) {
    double lo, hi;
    long long thr;
    int flags;
    bsc[r * 32 + lane] = row_phase1(raw + (long long)r * 2 * E, row0 + r, cap, E, L, io, status,
                                    lo, hi, thr, flags);
    if (lane == 0) {
      sc.lo[r] = lo;
      sc.hi[r] = hi;
      sc.t[r] = thr;
      sc.flags[r] = flags;
    }
  }
  __syncwarp();
  {
    double lo[1] = {lane < cap ? sc.lo[lane] : 0.0};
    double hi[1] = {lane < cap ? sc.hi[lane] : 0.0};
    const long long tt[1] = {lane < cap ? sc.t[lane] : 0};
    const bool bis[1] = {lane < cap && (sc.flags[lane] & 1)};
    const int iters = coupled_bisection<1>(lo, hi, tt, bis, cap);
    if (lane < cap) {
      sc.lo[lane] = lo[0];
      sc.hi[lane] = hi[0];
    }
    if (lane == 0) sc.iters = iters;
  }
  __syncwarp();
  for (int r = 0; r < cap; ++r)
    row_phase3(row0 + r, cap, E, L, io, bsc[r * 32 + lane], sc.lo[r], sc.hi[r], sc.flags[r],
               sc.iters, r);
}

// Mode R: the slot codebook [S][cap+1][E] plus optional diagnostics.
struct SlotIO {
  const int32_t* alloc;
  const double* eps;  // [S][cap][E] or null (deterministic)
  int32_t* cb;
  double* m_out;
  double* nu_out;
  double* margin_out;
  int32_t* iters_out;
  int E, cap;
  __device__ const int32_t* alloc_row(long long group) const { return alloc + group * E; }
  __device__ const double* eps_row(long long grow, long long, int) const {
    return eps ? eps + grow * E : nullptr;
  }
  __device__ void emit(long long grow, long long group, int j, int lane, int g, double m,
                       double nu, double margin, int iters) const {
    int32_t* book = cb + group * (cap + 1) * E;
    if (lane < E) {
      book[(long long)j * E + lane] = g;
      if (j == 1) book[lane] = 0;
      if (m_out) m_out[grow * E + lane] = m;
    }
    if (lane == 0) {
      if (nu_out) nu_out[grow] = nu;
      if (margin_out) margin_out[grow] = margin;
      if (iters_out && j == 1) iters_out[group] = iters;
    }
  }
  // one lane = one row (projection_lane.cuh): seats hT[e * 32], m_hat mT[e * 32]
  __device__ void emit_lane(long long grow, long long group, int j, const int* hT, int E_,
                            const double* mT, double nu, double margin, int iters) const {
    int32_t* book = cb + group * (cap + 1) * E;
    for (int e = 0; e < E; ++e) {
      book[(long long)j * E + e] = hT[e * 32];
      if (j == 1) book[e] = 0;
      if (m_out) m_out[grow * E + e] = mT[e * 32];
    }
    if (nu_out) nu_out[grow] = nu;
    if (margin_out) margin_out[grow] = margin;
    if (iters_out && j == 1) iters_out[group] = iters;
  }
};

template <typename RawT, int KE = 0>
__device__ void codebook_rows(const RawT* raw, const int32_t* alloc, const double* eps,
                              long long row0, int nrows, int cap, int E, int L, int32_t* cb,
                              double* m_out, double* nu_out, double* margin_out,
                              int32_t* iters_out, int32_t* status, RowScratch& sc,
                              unsigned long long* tr = nullptr) {
  const SlotIO io{alloc, eps, cb, m_out, nu_out, margin_out, iters_out, E, cap};
  codebook_rows_io<RawT, SlotIO, KE>(raw, row0, nrows, cap, E, L, io, status, sc, tr);
}

}  // namespace cyr
