// projection_lane.cuh — K3 for the throughput paths: ONE LANE PER ROW.
//
// The latency kernel and the standalone enforcer map one warp to one
// enforcement row (lane = eMBB user, projection.cuh) so a single slot's few
// rows finish fast.  For batches (Mode-R codebook batches, every Mode-T
// level) that mapping wastes lanes (E = 10 or 16 of 32) and spends most of
// its instructions on shuffles that emulate numpy's row sums.  Here a lane
// owns a whole row: the per-user loops run serially in registers, numpy's
// pairwise row sum is a plain loop in its exact association order, and the
// coupled bisection of a call (cap consecutive rows = cap consecutive lanes)
// is the same lanes = rows loop the warp version uses after its smem round
// trip.  Same float64 operations in the same order as projection.cuh (and
// the reference: enforcer.py:49-165, neural.py:144-183), hence the same bits.
//
// Per-warp shared memory, every array [E][32] (column = lane, so lanes
// access consecutive words): b / m_hat and the caps as doubles (the caps are
// read in every fill evaluation: one conversion per row instead of a global
// load + conversion per use) and the Huntington-Hill seat counts as ints.
#pragma once

#include "projection.cuh"

namespace cyr {

// numpy float64 add.reduce of term(0..n) (pairwise, 8 accumulators; n <= 128)
template <typename F>
__device__ __forceinline__ double np_sum_lane(int n, F term) {
  double acc;
  if (n < 8) {
    acc = 0.0;
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, term(i));
  } else {
    const int whole = n & ~7;
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = term(j);
    for (int blk = 8; blk < whole; blk += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], term(blk + j));
    acc = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                    __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (int i = whole; i < n; ++i) acc = __dadd_rn(acc, term(i));
  }
  return __dadd_rn(0.0, acc);
}

// One row held by one lane: b[e] at bT[e * 32] (this lane's column), caps
// from the allocation row (int32, shared by the call's rows), demand d.
struct LaneRow {
  double* bT;        // this lane's column of the warp's [E][32] array
  double* tT;        // scratch column (fill-evaluation terms; the HH seat arrays' space)
  const double* cT;  // caps (allocation row as doubles), same layout
  int E;
  double d;
  bool bis, degen, full;
  double lo, hi;
  mutable int evals;  // fill evaluations (CYR_TRACE profile only)
  __device__ __forceinline__ double b(int e) const { return bT[e * 32]; }
  __device__ __forceinline__ double c(int e) const { return cT[e * 32]; }
  __device__ __forceinline__ bool pos(int e) const { return b(e) > kMassFloor && c(e) > 0.0; }
};

// The terms go through the lane's scratch column so the quotient code exists
// once (a rolled loop) instead of once per unrolled slot of the pairwise sum
// at every call site: the lane kernel's hot loops had outgrown the
// instruction cache (stall_no_instruction 2.4 of 9.1 cycles per issue).
__device__ __forceinline__ bool fill_reaches_lane(const LaneRow& r, double x) {
  ++r.evals;
  const SharedDivisor sx = shared_divisor(x);  // one reciprocal for the row's E divisions
#pragma unroll 1
  for (int e = 0; e < r.E; ++e) r.tT[e * 32] = fmin(r.c(e), div_or_zero(r.b(e), sx));
  return np_sum_lane(r.E, [&](int e) { return r.tT[e * 32]; }) >= r.d;
}

// enforcer.py:57-89 (kl_setup of projection.cuh, one lane)
__device__ __forceinline__ void kl_setup_lane(LaneRow& r) {
  const double pos_cap = np_sum_lane(r.E, [&](int e) { return r.pos(e) ? r.c(e) : 0.0; });
  const bool active = r.d > 0.0;
  r.degen = active && (pos_cap < __dsub_rn(r.d, 1e-12));
  r.bis = active && !r.degen;
  r.full = r.bis && pos_cap <= r.d;
  r.lo = 0.0;
  r.hi = 0.0;
  if (r.bis) {
    double lo = CUDART_INF;
    for (int e = 0; e < r.E; ++e)
      if (r.pos(e)) lo = fmin(lo, __ddiv_rn(r.b(e), fmax(r.c(e), 1e-300)));
    const double hi = __ddiv_rn(np_sum_lane(r.E, [&](int e) { return r.b(e); }), r.d);
    r.lo = fmin(lo, hi);
    r.hi = hi;
  }
}

// Water-level estimate (any summation order: only a starting point for the
// exact threshold search) — water_level of projection.cuh.
__device__ __forceinline__ double water_level_lane(const LaneRow& r) {
  if (r.full) return r.lo;  // all users capped (water_level of projection.cuh)
  double nu = r.hi;
  unsigned prev = 0xffffffffu;
  for (int it = 0; it <= r.E; ++it) {
    unsigned mask = 0;
    double cc = 0.0, bu = 0.0;
    for (int e = 0; e < r.E; ++e) {
      const double b = r.b(e), c = r.c(e);
      const bool capped = b > kMassFloor && c > 0.0 && b >= nu * c;
      mask |= capped ? 1u << e : 0u;
      if (capped) cc += c;
      else bu += b;
    }
    if (mask == prev) break;
    prev = mask;
    const double den = r.d - cc;
    if (den <= 0.0) {
      nu = CUDART_INF;
      for (int e = 0; e < r.E; ++e)
        if ((mask >> e) & 1u) nu = fmin(nu, r.b(e) / fmax(r.c(e), 1e-300));
      break;
    }
    nu = bu / den;
  }
  if (!(nu > 0.0) || isinf(nu)) nu = sqrt(r.lo) * sqrt(r.hi);
  return nu;
}

// Exact fill threshold (fill_threshold of projection.cuh, one lane): gallop
// from the water level, then halve.  One evaluation site (a state machine)
// keeps the loop's code small.
__device__ __forceinline__ long long fill_threshold_lane(const LaneRow& r, double x0) {
  constexpr long long kInf = 0x7ff0000000000000ll;
  const long long a = __double_as_longlong(x0);
  long long lo = 0, hi = 0, step = 1, cand = a;
  int ph = 0;  // 0 first probe, 1 gallop up, 2 gallop down, 3 halve
#pragma unroll 1
  for (;;) {
    const bool ok = fill_reaches_lane(r, __longlong_as_double(cand));
    if (ph == 0) {
      if (ok) { lo = a; ph = 1; } else { hi = a; ph = 2; }
    } else if (ph == 1) {
      if (ok) { lo = cand; step <<= 1; } else { hi = cand; ph = 3; }
    } else if (ph == 2) {
      if (ok) { lo = cand; ph = 3; } else { hi = cand; step <<= 1; }
    } else {
      if (ok) lo = cand; else hi = cand;
    }
    if (ph == 1) {
      cand = lo + step;
      if (cand >= kInf) { hi = kInf; ph = 3; }
    } else if (ph == 2) {
      cand = hi - step;
      if (cand <= 0) { lo = 0; ph = 3; }
    }
    if (ph == 3) {
      if (hi - lo <= 1) break;
      cand = lo + ((hi - lo) >> 1);
    }
  }
  return lo;
}

// m_hat into bT (overwriting b) and the row's nu (kl_finish, enforcer.py:98-114)
__device__ __forceinline__ double kl_finish_lane(LaneRow& r) {
  if (r.bis) {
    const double nu = __dmul_rn(__dsqrt_rn(r.lo), __dsqrt_rn(r.hi));
    const SharedDivisor snu = shared_divisor(nu);
    for (int e = 0; e < r.E; ++e) r.bT[e * 32] = fmin(r.c(e), div_or_zero(r.b(e), snu));
    return nu;
  }
  if (r.degen) {
    const double slack =
        __dsub_rn(r.d, np_sum_lane(r.E, [&](int e) { return r.pos(e) ? r.c(e) : 0.0; }));
    const double spare = np_sum_lane(r.E, [&](int e) { return r.pos(e) ? 0.0 : r.c(e); });
    for (int e = 0; e < r.E; ++e) {
      double fill = r.pos(e) ? r.c(e) : 0.0;
      if (spare > 0.0 && slack > 0.0 && !r.pos(e))
        fill = div_or_zero(__dmul_rn(r.c(e), slack), spare);
      r.bT[e * 32] = fill;  // in place: pos(e) of later users reads their own b
    }
    return 0.0;
  }
  for (int e = 0; e < r.E; ++e) r.bT[e * 32] = 0.0;
  return 0.0;
}

// sqrt(max(a(a+1), 1)) of seat a = 0 .. kSeatTab-1, the divisor of the
// reference's seat priority (enforcer.py:150-154): built once per device by
// seat_table_kernel with the same __dsqrt_rn expression as seat_prio, so a
// table lookup is bit-identical to computing it (one division per priority
// instead of a division and a square root).
// The table also holds each divisor's correctly rounded reciprocal, so a
// priority is a Markstein quotient (SharedDivisor) instead of a division.
constexpr int kSeatTab = 1024;
static __device__ double2 g_seat_div[kSeatTab];  // {sqrt(max(a(a+1), 1)), RN(1 / that)}

static __global__ void seat_table_kernel() {
  for (int a = threadIdx.x; a < kSeatTab; a += blockDim.x) {
    const double x = (double)a;
    const double d = __dsqrt_rn(fmax(__dmul_rn(x, __dadd_rn(x, 1.0)), 1.0));
    g_seat_div[a] = make_double2(d, __drcp_rn(d));
  }
}

__device__ __forceinline__ double seat_prio_tab(double m, int seat) {
  if (seat < kSeatTab) {
    const double2 t = g_seat_div[seat];
    return div_or_zero(m, shared_divisor(t.x, t.y));
  }
  return seat_prio(m, seat);
}

// Huntington-Hill seats for m = mT[e * 32], caps cT; seats into hT[e * 32]
// (hh_row of projection.cuh, one lane).  Returns the near-tie margin.  nT
// caches each user's seat count once per row: cnt = ceil(cap) when the user
// has positive mass and cnt >= 1, else -cnt - 1.
__device__ __forceinline__ double hh_lane(const double* mT, const double* cT, int E, long long want,
                                          int* hT, int* nT, int* steps_out = nullptr) {
  auto m = [&](int e) { return mT[e * 32]; };
  for (int e = 0; e < E; ++e) {
    const int c = (int)ceil(cT[e * 32]);
    nT[e * 32] = (m(e) > 0.0 && c >= 1) ? c : -c - 1;
  }
  auto cnt = [&](int e) {
    const int v = nT[e * 32];
    return v >= 1 ? v : -v - 1;
  };
  auto posu = [&](int e) { return nT[e * 32] >= 1; };
  double margin = CUDART_INF;
  for (int e = 0; e < E; ++e) hT[e * 32] = 0;
  if (want <= 0) return margin;
  int n0 = 0;
  for (int e = 0; e < E; ++e) n0 += posu(e) ? 1 : 0;

  if (want <= n0) {  // phase 0: first seats by mass (desc), user index (asc)
    int last = -1, next = -1;
    for (int e = 0; e < E; ++e) {
      if (!posu(e)) continue;
      const double me = m(e);
      int rank = 0;
      for (int f = 0; f < E; ++f)
        if (posu(f) && precedes(m(f), f, me, e)) ++rank;
      if (rank < want) hT[e * 32] = 1;
      if (rank == want - 1) last = e;
      if (rank == want) next = e;
    }
    if (last >= 0 && next >= 0) margin = div_or_zero(__dsub_rn(m(last), m(next)), m(last));
    return margin;
  }

  const long long r1 = want - n0;
  long long p1 = 0;
  for (int e = 0; e < E; ++e) p1 += posu(e) ? cnt(e) - 1 : 0;
  if (r1 <= p1) {  // phase 1: exact top-r1 by exchange from the lambda = 1 guess
    long long total = 0;
    for (int e = 0; e < E; ++e) {
      int h = 0;
      if (posu(e)) {
        const double me = m(e);
        int g = (int)floor(me);
        if (g >= 1 && (double)g * (double)(g + 1) > me * me) g -= 1;
        h = max(0, min(g, cnt(e) - 1));
      }
      hT[e * 32] = h;
      total += h;
    }
    const long long guard = 256 + 4 * r1;
    for (long long step = 0; step < guard; ++step) {
      // best add candidate (first in order) and worst held seat (last)
      bool oka = false, okd = false;
      double pa = 0.0, pd = 0.0;
      int la = 0, ld = 0;
      for (int e = 0; e < E; ++e) {
        if (!posu(e)) continue;
        const int h = hT[e * 32];
        const double me = m(e);
        if (h + 1 <= cnt(e) - 1) {
          const double p = seat_prio_tab(me, h + 1);
          if (!oka || precedes(p, e, pa, la)) {
            pa = p;
            la = e;
            oka = true;
          }
        }
        if (h >= 1) {
          const double p = seat_prio_tab(me, h);
          if (!okd || precedes(pd, ld, p, e)) {
            pd = p;
            ld = e;
            okd = true;
          }
        }
      }
      if (total < r1) {
        hT[la * 32] += 1;
        ++total;
      } else if (total > r1) {
        hT[ld * 32] -= 1;
        --total;
      } else if (oka && okd && precedes(pa, la, pd, ld)) {
        hT[la * 32] += 1;
        hT[ld * 32] -= 1;
      } else {
        if (oka && okd) margin = div_or_zero(__dsub_rn(pd, pa), pd);
        if (steps_out) *steps_out = (int)step + 1;
        break;
      }
    }
    for (int e = 0; e < E; ++e) hT[e * 32] = posu(e) ? 1 + hT[e * 32] : 0;
    return margin;
  }

  // every positive-mass user full; zero-mass users: first seats in index
  // order (phase 2), then later seats user by user (phase 3)
  long long r2 = r1 - p1;
  int nz = 0;
  for (int e = 0; e < E; ++e) {
    const bool zu = !(m(e) > 0.0) && cnt(e) >= 1;
    int g = posu(e) ? cnt(e) : 0;
    if (zu) {
      if (nz < r2) g += 1;
      ++nz;
    }
    hT[e * 32] = g;
  }
  long long r3 = r2 - nz;
  for (int e = 0; e < E && r3 > 0; ++e) {
    const bool zu = !(m(e) > 0.0) && cnt(e) >= 1;
    if (!zu) continue;
    const long long add = min((long long)(cnt(e) - 1), r3);
    hT[e * 32] += (int)add;
    r3 -= add;
  }
  return margin;
}

// Per-warp scratch for up to 32 rows of E users: bT, cT (double), hT and
// nT (int), each [E][32].
__host__ __device__ constexpr size_t lane_scratch_bytes(int E) {
  return (size_t)E * 32 * (2 * sizeof(double) + 2 * sizeof(int));
}

// Rows row0 .. row0 + nrows of this warp (whole calls of `cap` rows, lane
// r = local row r).  IO: alloc_row(group), eps_row(grow, group, j) and
// emit_lane(grow, group, j, hT, E, mT, nu, margin, iters) (one lane).
// CYR_TRACE=1 phase profile of the lane mapping (prof != null): per warp,
// clock64 cycles of each phase summed into prof[0..7] (head, setup, water
// level, threshold, coupled loop, finish, Huntington-Hill, emit), warps in
// prof[8].  Diagnostics only (system-scope atomics on mapped memory).
#ifndef CYR_HEAD_UNROLL
#define CYR_HEAD_UNROLL 1
#endif
constexpr int kHeadUnroll = CYR_HEAD_UNROLL;  // head loop unroll (A/B)
// KE > 0: the user count as a compile-time constant (every per-user loop
// has a known trip count); 0: runtime E.
template <typename RawT, typename IO, int KE = 0>
__device__ void codebook_rows_lane(const RawT* raw, long long row0, int nrows, int cap, int E_rt,
                                   int L, const IO& io, int32_t* status, unsigned char* scratch,
                                   unsigned long long* prof = nullptr) {
  const int E = KE > 0 ? KE : E_rt;
  const int lane = threadIdx.x & 31;
  long long tp = prof ? clock64() : 0;
  auto mark = [&](int k) {
    if (prof) {
      __syncwarp();
      const long long now = clock64();
      if (lane == 0) atomicAdd(prof + k, (unsigned long long)(now - tp));
      tp = now;
    }
  };
  const size_t plane = (size_t)E * 32;  // elements of one [E][32] array
  double* bT = reinterpret_cast<double*>(scratch) + lane;
  double* cT = bT + plane;
  int* hT = reinterpret_cast<int*>(scratch + 2 * plane * sizeof(double)) + lane;
  int* nT = hT + plane;
  const bool live = lane < nrows;
  const long long grow = row0 + (live ? lane : 0);
  const long long group = grow / cap;
  const int j = (int)(grow % cap) + 1;
  LaneRow r;
  r.bT = bT;
  r.cT = cT;
  r.tT = reinterpret_cast<double*>(scratch + 2 * plane * sizeof(double)) + lane;  // = hT/nT space
  if (live) {
    const int32_t* n = io.alloc_row(group);
    for (int e = 0; e < E; ++e) cT[e * 32] = (double)__ldg(n + e);
  }
  r.E = E;
  r.d = (double)((long long)j * L);
  r.bis = r.degen = r.full = false;
  r.lo = r.hi = 0.0;
  r.evals = 0;
  long long thr = 0;
  if (live) {
    // head (neural.py:144-165, sac.py:348-355) and action_to_scs (neural.py:181-183)
    const RawT* rr = raw + (long long)lane * 2 * E;
    const double* eps = io.eps_row(grow, group, j);
#pragma unroll (kHeadUnroll)
    for (int e = 0; e < E; ++e) {
      const double mu = (double)rr[e];
      const double ls = fmin(fmax((double)rr[E + e], kLogSigmaMin), kLogSigmaMax);
      const double a = eps ? tanh(__dadd_rn(mu, __dmul_rn(exp(ls), eps[e]))) : tanh(mu);
      bT[e * 32] = __dmul_rn(__dmul_rn(__dadd_rn(a, 1.0), 0.5), r.c(e));
    }
  }
  mark(0);
  double x0 = 0.0;
  if (live) {
    const double capsum = np_sum_lane(E, [&](int e) { return r.c(e); });  // enforcer.py:64
    if (r.d > capsum) set_status(status, CYR_INFEASIBLE);
    kl_setup_lane(r);
  }
  mark(1);
  if (live && r.bis) x0 = water_level_lane(r);
  mark(2);
  if (live && r.bis) thr = fill_threshold_lane(r, x0);
  mark(3);
  // the coupled loop of every call of the warp at once (lanes = rows)
  double lo[1] = {r.lo}, hi[1] = {r.hi};
  const long long tt[1] = {thr};
  const bool bis[1] = {live && r.bis};
  const int iters = coupled_bisection<1, true>(lo, hi, tt, bis, cap);
  r.lo = lo[0];
  r.hi = hi[0];
  mark(4);
  double nu = 0.0, margin = 0.0;
  if (live) nu = kl_finish_lane(r);
  mark(5);
  int hh_steps = 0;
  if (live) margin = hh_lane(bT, cT, E, (long long)j * L, hT, nT, prof ? &hh_steps : nullptr);
  mark(6);
  if (live) io.emit_lane(grow, group, j, hT, E, bT, nu, margin, iters);
  mark(7);
  if (prof) {  // event counts summed over the warp's live rows
    unsigned long long ev = live ? (unsigned long long)r.evals : 0ull;
    unsigned long long hs = live ? (unsigned long long)hh_steps : 0ull;
    for (int o = 16; o > 0; o >>= 1) {
      ev += __shfl_xor_sync(0xffffffffu, ev, o);
      hs += __shfl_xor_sync(0xffffffffu, hs, o);
    }
    const unsigned nlive = (unsigned)__popc(__ballot_sync(0xffffffffu, live));
    int emax = live ? r.evals : 0, hmax = live ? hh_steps : 0;
    for (int o = 16; o > 0; o >>= 1) {
      emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
      hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
    }
    if (live) {  // histogram of fill evaluations per row: bins 1 .. 11, 12+ (prof[16..27])
      const int bin = min(max(r.evals, 1), 12) - 1;
      atomicAdd(prof + 16 + bin, 1ull);
    }
    if (lane == 0) {
      atomicAdd(prof + 8, 1ull);
      atomicAdd(prof + 9, ev);
      atomicAdd(prof + 10, hs);
      atomicAdd(prof + 11, (unsigned long long)nlive);
      atomicAdd(prof + 12, (unsigned long long)iters);
      atomicAdd(prof + 13, (unsigned long long)emax);  // warp's slowest lane: what the warp runs
      atomicAdd(prof + 14, (unsigned long long)hmax);
    }
  }
}

}  // namespace cyr
