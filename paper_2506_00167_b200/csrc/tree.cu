// tree.cu — K1: Mode-R arrival-tree expansion / node-state kernel.
//
// No reference function builds the tree.  What it
// materialises is the composition of reference steps for EVERY admissible
// URLLC arrival pattern of a slot: the applied puncture rows are codebook
// columns looked up per mini-slot (engine.py:230) and a user's punctured
// total is their sum (engine.py:240-241, phy.py:201).
//
// Layout: per slot, levels t = 1..M in BFS order; level t holds (cap+1)^t
// nodes; the children of node p of level t-1 are p*(cap+1) + k, k = 0..cap,
// so the children of a contiguous parent range are one contiguous run.
// A node record is the per-user cumulative puncture count as int16, packed:
// Ep = roundup(E, 2) lanes = W 4-byte words (20 B at E = 10, 8 B at E = 4,
// 32 B at E = 16).  Only the algorithmic bytes reach HBM (the earlier
// 16-byte-granule padding wrote 32 B records at E = 10: 60 % more).
//
// B200 design (HBM-write-bound): a persistent grid; each CTA owns a
// contiguous range of work items = (slot, level, block of NP parents), so
// the per-slot setup — the codebook columns in registers and the 3-digit
// suffix table T3 in shared memory — is built once per slot a CTA touches,
// not once per item.  Codebook column 0 is the all-zero vector
// (engine.py:112), so leading zero digits add nothing and a parent's state
// is T3[p mod R^3] + T3[p div R^3] (+ T3[...] for deeper trees): two
// shared-memory lookups instead of a per-digit divide-and-add loop.  Each
// child is one packed 16-bit vector add (__vadd2) per word into a
// shared-memory staging buffer laid out exactly like the child run in HBM
// (shifted so smem and global addresses agree mod 16).  One thread writes
// the run's 16-byte-aligned body with a single TMA bulk store
// (cp.async.bulk.global.shared::cta, SASS UBLKCP); the at most 3 + 3 words
// of unaligned head and tail go out as plain stores.  A ring of kStages
// staging buffers with ONE CTA barrier per item lets the next items'
// compute overlap the previous stores.  A codebook whose column 0 is not
// zero falls back to the per-digit sum.
#include "cyrus_internal.cuh"
#include "cyrus_b200.h"

#include <algorithm>
#include <cstdlib>

namespace cyr {

constexpr int kTreeThreads = 128;  // parents per full work item (= threads per CTA)
constexpr int kStages = 3;         // staging buffers per CTA
constexpr int kMaxLevels = 16;

struct TreeParams {
  const int32_t* codebook;
  int16_t* out;
  int S, E, cap, M;
  int words;                         // 4-byte words per record (Ep / 2)
  int np_item;                       // parents per work item (<= kTreeThreads)
  int r3;                            // (cap+1)^3
  unsigned r3_magic;                 // floor(q / r3) == __umulhi(q, r3_magic) in range
  long long nodes_per_slot;
  int blocks_per_slot;
  int level_blocks[kMaxLevels + 1];  // prefix over parent levels t = 0..M-1
  long long level_parents[kMaxLevels];
  long long child_off[kMaxLevels];   // node offset of level t+1 within a slot
  // leaf scoring, SCORE instantiation only
  const int32_t* alloc;              // [S][E] allocations n_e
  const double* margin;              // [S][E] threshold-decoder margins
  const double* prob;                // [M][R] admitted-count probabilities per mini-slot
  int N;                             // total SCs (reward denominator)
  uint32_t* leaf_ok;                 // [S][R^M] decoding-user bitmask, or null
  double* partial;                   // [S][leaf items][2]: sum w*lost, sum w*goodput
};

__host__ __device__ __forceinline__ size_t tree_stage_bytes(int np, int R, int words) {
  return ((size_t)np * R * words * 4 + 15) / 16 * 16 + 16;  // + 16: the mod-16 shift
}

__device__ __forceinline__ uint4 vadd16(uint4 a, uint4 b) {
  return make_uint4(__vadd2(a.x, b.x), __vadd2(a.y, b.y), __vadd2(a.z, b.z), __vadd2(a.w, b.w));
}

// Leaf epilogue (SCORE): the threshold decoder of every user at every leaf
// (phy.py:73-80 via decode_user, phy.py:196-198): ok_e = n_e <= 0 or
// cum_e <= margin_e * (M * n_e).  cum is an integer, so the float64 bound
// becomes an exact int16 bound (floor), and a packed signed compare
// (__vcmples2) decides two users per instruction.  lost = sum of n_e over
// failing users (core.py:132-146: r = -lost / N), goodput = sum n_e - lost.
// Each leaf's weight is the product over mini-slots of the admitted-count
// probability of its digit; the CTA reduces sum(w * lost) and
// sum(w * goodput) deterministically into one partial per work item.
__device__ __forceinline__ unsigned lane_bits(unsigned m) {  // 0xffff lanes -> 2 bits
  return (m & 1u) | ((m >> 15) & 2u);
}

template <int CH, int R, bool SCORE>  // CH: 16-byte register granules per record; R = cap + 1
__global__ void __launch_bounds__(kTreeThreads) tree_kernel(const TreeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int NP = p.np_item;
  const int W = p.words;
  const size_t stage_bytes = tree_stage_bytes(NP, R, W);
  const int r3 = p.r3;
  uint4* t3 = reinterpret_cast<uint4*>(smem + kStages * stage_bytes);  // [r3][CH], per slot
  int16_t* bookw = reinterpret_cast<int16_t*>(t3 + (size_t)r3 * CH);   // [R][CH*8]
  // SCORE: per-user int16 bounds and allocations as packed granules, leaf-digit
  // probabilities, and the CTA reduction scratch
  int16_t* boundw = bookw + R * CH * 8;                 // [CH*8]
  int16_t* allocw = boundw + CH * 8;                    // [CH*8]
  double* probs = reinterpret_cast<double*>(allocw + CH * 8);  // [M][R]
  double* red = probs + kMaxLevels * R;                 // [kTreeThreads / 32][2]
  const int tid = threadIdx.x;
  const int items = p.S * p.blocks_per_slot;  // host-checked to fit in int
  // this CTA's contiguous item range
  const int chunk = (items + gridDim.x - 1) / gridDim.x;
  const int w_begin = blockIdx.x * chunk;
  const int w_end = min(items, w_begin + chunk);
  int cur_s = -1;
  uint4 col[R][CH];
  bool zero0 = true;
  int it = 0;
  for (int w = w_begin; w < w_end; ++w, ++it) {
    const int s = w / p.blocks_per_slot;
    const int bw = w - s * p.blocks_per_slot;
    int t = 0;
    while (bw >= p.level_blocks[t + 1]) ++t;
    const int p0 = (bw - p.level_blocks[t]) * NP;
    const int np = (int)min((long long)NP, p.level_parents[t] - p0);

    if (s != cur_s) {  // per-slot setup (uniform branch)
      __syncthreads();  // every thread is done with the previous slot's tables
      // the slot's codebook as packed int16 granules, then every thread keeps
      // the cap+1 columns in registers
      const int32_t* cb = p.codebook + (long long)s * R * p.E;
      for (int idx = tid; idx < R * CH * 8; idx += kTreeThreads) {
        const int k = idx / (CH * 8), e = idx % (CH * 8);
        bookw[idx] = (int16_t)((e < p.E) ? cb[k * p.E + e] : 0);
      }
      if constexpr (SCORE) {
        for (int e = tid; e < CH * 8; e += kTreeThreads) {
          int bound = 32767, n = 0;  // padding lanes: always "ok", no SCs
          if (e < p.E) {
            n = p.alloc[(long long)s * p.E + e];
            if (n > 0) {
              const double rhs = __dmul_rn(p.margin[(long long)s * p.E + e], (double)(p.M * n));
              bound = rhs >= 32767.0 ? 32767 : (rhs < 0.0 ? -1 : (int)floor(rhs));
            }
          }
          boundw[e] = (int16_t)bound;
          allocw[e] = (int16_t)(n > 0 ? n : 0);
        }
        for (int idx = tid; idx < p.M * R; idx += kTreeThreads) probs[idx] = p.prob[idx];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int c = 0; c < CH; ++c) col[k][c] = reinterpret_cast<const uint4*>(bookw)[k * CH + c];
      zero0 = true;
#pragma unroll
      for (int c = 0; c < CH; ++c)
        zero0 = zero0 && (col[0][c].x | col[0][c].y | col[0][c].z | col[0][c].w) == 0u;
      // suffix table of every 3-digit suffix
      for (int x = tid; x < r3; x += kTreeThreads) {
        const int d0 = x % R, d1 = (x / R) % R, d2 = x / (R * R);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          uint4 v = make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const uint4 ck = col[k][c];
            if (d0 == k) v = vadd16(v, ck);
            if (d1 == k) v = vadd16(v, ck);
            if (d2 == k) v = vadd16(v, ck);
          }
          t3[x * CH + c] = v;
        }
      }
      __syncthreads();
      cur_s = s;
    }

    // this item's child run in HBM: bytes [gbeg, gend) from p.out
    const long long first = (long long)s * p.nodes_per_slot + p.child_off[t] + (long long)p0 * R;
    const long long gbeg = first * W * 4;
    const int shift = (int)(gbeg & 15);  // smem copy sits at the same address mod 16
    uint32_t* stw =
        reinterpret_cast<uint32_t*>(smem + (size_t)(it % kStages) * stage_bytes + shift);
    double acc_lost = 0.0, acc_good = 0.0;  // SCORE: this thread's weighted leaf sums

    if (tid < np) {
      uint4 cum[CH];
      unsigned q = (unsigned)(p0 + tid);
      if (zero0) {
        const unsigned hi = __umulhi(q, p.r3_magic);
        const unsigned lo = q - hi * (unsigned)r3;
#pragma unroll
        for (int c = 0; c < CH; ++c) cum[c] = t3[lo * CH + c];
        if (t > 3) {  // 4..6 parent digits: one more suffix lookup (7..9: two)
          const unsigned hh = __umulhi(hi, p.r3_magic);
          const unsigned hl = hi - hh * (unsigned)r3;
#pragma unroll
          for (int c = 0; c < CH; ++c) cum[c] = vadd16(cum[c], t3[hl * CH + c]);
          if (t > 6)
#pragma unroll
            for (int c = 0; c < CH; ++c) cum[c] = vadd16(cum[c], t3[hh * CH + c]);
        }
      } else {  // general codebook: per-digit sum
#pragma unroll
        for (int c = 0; c < CH; ++c) cum[c] = make_uint4(0, 0, 0, 0);
        for (int d = 0; d < t; ++d) {
          const unsigned nq = q / (unsigned)R;
          const int k = (int)(q - nq * (unsigned)R);
          q = nq;
#pragma unroll
          for (int kk = 0; kk < R; ++kk)
            if (kk == k)
#pragma unroll
              for (int c = 0; c < CH; ++c) cum[c] = vadd16(cum[c], col[kk][c]);
        }
      }
      uint32_t* dst = stw + (size_t)tid * R * W;
      if (W == CH * 4) {  // E a multiple of 8: whole granules (shift is 0, 16-B aligned)
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int c = 0; c < CH; ++c)
            reinterpret_cast<uint4*>(dst)[k * CH + c] = vadd16(cum[c], col[k][c]);
      } else {
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const uint4 v = vadd16(cum[c], col[k][c]);
            uint32_t* d = dst + k * W + 4 * c;
            if (4 * c + 0 < W) d[0] = v.x;
            if (4 * c + 1 < W) d[1] = v.y;
            if (4 * c + 2 < W) d[2] = v.z;
            if (4 * c + 3 < W) d[3] = v.w;
          }
      }
      if constexpr (SCORE) {
        if (t == p.M - 1) {  // children are leaves
          double wq = 1.0;   // parent weight: its M-1 digits, first mini-slot first
          unsigned x = (unsigned)(p0 + tid), div = 1;
          for (int d = 1; d < p.M - 1; ++d) div *= (unsigned)R;
          for (int d = 0; d < p.M - 1; ++d) {
            const unsigned dig = x / div;
            x -= dig * div;
            div /= (unsigned)R;
            wq = __dmul_rn(wq, probs[d * R + dig]);
          }
          const uint4* bw4 = reinterpret_cast<const uint4*>(boundw);
          const uint4* aw4 = reinterpret_cast<const uint4*>(allocw);
          unsigned tot = 0;
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const uint4 a = aw4[c];
            tot += (a.x & 0xffffu) + (a.x >> 16) + (a.y & 0xffffu) + (a.y >> 16) +
                   (a.z & 0xffffu) + (a.z >> 16) + (a.w & 0xffffu) + (a.w >> 16);
          }
          const long long leaf0 = (long long)s * p.level_parents[p.M - 1] * R +
                                  (long long)(p0 + tid) * R;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            unsigned okbits = 0, lost2 = 0;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              const uint4 v = vadd16(cum[c], col[k][c]), b = bw4[c], a = aw4[c];
              const unsigned m0 = __vcmples2(v.x, b.x), m1 = __vcmples2(v.y, b.y);
              const unsigned m2 = __vcmples2(v.z, b.z), m3 = __vcmples2(v.w, b.w);
              okbits |= (lane_bits(m0) | lane_bits(m1) << 2 | lane_bits(m2) << 4 |
                         lane_bits(m3) << 6) << (8 * c);
              lost2 = __vadd2(lost2, __vadd2(__vadd2(~m0 & a.x, ~m1 & a.y),
                                             __vadd2(~m2 & a.z, ~m3 & a.w)));
            }
            const unsigned lost = (lost2 & 0xffffu) + (lost2 >> 16);
            const double wgt = __dmul_rn(wq, probs[(p.M - 1) * R + k]);
            acc_lost = __fma_rn(wgt, (double)lost, acc_lost);
            acc_good = __fma_rn(wgt, (double)(tot - lost), acc_good);
            if (p.leaf_ok)
              p.leaf_ok[leaf0 + k] = okbits & (p.E >= 32 ? 0xffffffffu : ((1u << p.E) - 1u));
          }
        }
      }
    }
    fence_proxy_async_smem();  // generic smem writes -> visible to the bulk-copy proxy
    if constexpr (SCORE) {
      if (t == p.M - 1) {  // deterministic CTA reduction -> this item's partial
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          acc_lost += __shfl_down_sync(0xffffffffu, acc_lost, off);
          acc_good += __shfl_down_sync(0xffffffffu, acc_good, off);
        }
        if ((tid & 31) == 0) {
          red[(tid >> 5) * 2] = acc_lost;
          red[(tid >> 5) * 2 + 1] = acc_good;
        }
        __syncthreads();
        if (tid == 0) {
          double l = 0.0, g = 0.0;
          for (int wi = 0; wi < kTreeThreads / 32; ++wi) {
            l += red[wi * 2];
            g += red[wi * 2 + 1];
          }
          const long long item = (long long)s * (p.level_blocks[p.M] - p.level_blocks[p.M - 1]) +
                                 (bw - p.level_blocks[p.M - 1]);
          p.partial[item * 2] = l;
          p.partial[item * 2 + 1] = g;
        }
      }
    }
    // Before the barrier, the store issued kStages-1 items ago must have read
    // its stage: that is the buffer the NEXT item writes after the barrier.
    if (tid == 0) bulk_wait_read<kStages - 2>();
    __syncthreads();
    {
      // body [a16, b16): one bulk store; head [gbeg, a16) and tail [b16, gend):
      // at most 3 words each, plain stores (neighbouring items own the other
      // bytes of those granules)
      const long long gend = gbeg + (long long)np * R * W * 4;
      long long a16 = (gbeg + 15) & ~15ll, b16 = gend & ~15ll;
      if (b16 < a16) a16 = b16 = gend;  // shorter than one granule: all plain
      unsigned char* ob = reinterpret_cast<unsigned char*>(p.out);
      const unsigned char* sb = reinterpret_cast<const unsigned char*>(stw);
      if (tid == 0) {
        if (b16 > a16) bulk_s2g(ob + a16, sb + (a16 - gbeg), (uint32_t)(b16 - a16));
        bulk_commit();  // one group per item (possibly empty): the ring parity stays exact
      }
      if (tid >= 32 && tid < 35) {  // head words
        const long long g = gbeg + 4 * (tid - 32);
        if (g < a16)
          *reinterpret_cast<uint32_t*>(ob + g) = *reinterpret_cast<const uint32_t*>(sb + (g - gbeg));
      } else if (tid >= 64 && tid < 67) {  // tail words
        const long long g = b16 + 4 * (tid - 64);
        if (g >= a16 && g < gend)
          *reinterpret_cast<uint32_t*>(ob + g) = *reinterpret_cast<const uint32_t*>(sb + (g - gbeg));
      }
    }
  }
  if (tid == 0) bulk_wait_all();
}

// expected values per slot from the per-item partials, in item order
__global__ void tree_score_reduce_kernel(const double* __restrict__ partial, int items, int S,
                                         int N, double* __restrict__ expect) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  double l = 0.0, g = 0.0;
  for (int i = 0; i < items; ++i) {
    l += partial[((long long)s * items + i) * 2];
    g += partial[((long long)s * items + i) * 2 + 1];
  }
  expect[s * 3] = -l / (double)N;  // E[r] (core.py:132-146)
  expect[s * 3 + 1] = g;           // E[goodput SCs] (core.py:149-153)
  expect[s * 3 + 2] = l;           // E[lost SCs]
}

template <int CH, int R, bool SCORE>
int launch_tree_t(const TreeParams& p, int sm_count, cudaStream_t stream) {
  const size_t smem = kStages * tree_stage_bytes(p.np_item, R, p.words) +
                      (size_t)p.r3 * CH * 16 + (size_t)R * CH * 16 +
                      (SCORE ? 2 * (size_t)CH * 16 + (size_t)kMaxLevels * R * 8 +
                                   (kTreeThreads / 32) * 16
                             : 0);
  if (smem > 227 * 1024) return CYR_UNSUPPORTED;
  auto kern = tree_kernel<CH, R, SCORE>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return CYR_CUDA_ERROR;
  const long long items = (long long)p.S * p.blocks_per_slot;
  const int fit = (int)std::max<size_t>(1, (227 * 1024) / (smem + 1024));
  // 4 resident CTAs per SM (sweep, bench workload, 128-parent items: 3 / 4 / 5
  // per SM = 368 / 301 / 353 us; more concurrent write streams lose HBM
  // efficiency, as in the pure-write microbenchmark, profiles/r01_write_patterns.txt)
  int per_sm = std::min(fit, 4);
  static const int per_sm_env = [] {  // CYR_TREE_PER_SM: resident CTAs per SM (A/B)
    const char* e = getenv("CYR_TREE_PER_SM");
    return e ? atoi(e) : 0;
  }();
  if (per_sm_env > 0) per_sm = std::min(per_sm_env, fit);
  const long long grid = std::min<long long>(items, (long long)sm_count * per_sm);
  kern<<<(unsigned)grid, kTreeThreads, smem, stream>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

template <int CH, bool SCORE>
int launch_tree_r(const TreeParams& p, int sm_count, cudaStream_t stream) {
  switch (p.cap + 1) {
    case 2: return launch_tree_t<CH, 2, SCORE>(p, sm_count, stream);
    case 3: return launch_tree_t<CH, 3, SCORE>(p, sm_count, stream);
    case 4: return launch_tree_t<CH, 4, SCORE>(p, sm_count, stream);
    case 5: return launch_tree_t<CH, 5, SCORE>(p, sm_count, stream);
    case 6: return launch_tree_t<CH, 6, SCORE>(p, sm_count, stream);
    case 7: return launch_tree_t<CH, 7, SCORE>(p, sm_count, stream);
    case 8: return launch_tree_t<CH, 8, SCORE>(p, sm_count, stream);
    case 9: return launch_tree_t<CH, 9, SCORE>(p, sm_count, stream);
    default: return CYR_UNSUPPORTED;
  }
}

template <bool SCORE>
int launch_tree_ch(const TreeParams& p, int sm_count, cudaStream_t stream) {
  switch ((p.words * 2 + 7) / 8) {
    case 1: return launch_tree_r<1, SCORE>(p, sm_count, stream);
    case 2: return launch_tree_r<2, SCORE>(p, sm_count, stream);
    case 3: return launch_tree_r<3, SCORE>(p, sm_count, stream);
    default: return launch_tree_r<4, SCORE>(p, sm_count, stream);
  }
}

// geometry of the level-synchronous work items (shared by both entry points)
int tree_params(TreeParams& p, const int32_t* codebook, int S, int E, int cap, int M,
                int16_t* out, int sm_count) {
  if (E < 1 || E > kMaxUsers || cap < 1 || M < 1 || M > 10) return CYR_BAD_ARG;
  if (cap + 1 > 9) return CYR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return CYR_BAD_ARG;
  p.codebook = codebook;
  p.out = out;
  p.S = S;
  p.E = E;
  p.cap = cap;
  p.M = M;
  p.words = (E + 1) / 2;
  const long long R = cap + 1;
  p.r3 = (int)(R * R * R);
  // ceil(2^32 / r3): floor(q * magic / 2^32) == floor(q / r3) while
  // q * (magic * r3 - 2^32) < 2^32, i.e. for every q < 2^32 / r3
  p.r3_magic = (unsigned)((0x100000000ull + p.r3 - 1) / p.r3);
  long long top = 1;
  for (int t = 0; t < M - 1; ++t) top *= R;
  if (top * p.r3 >= (1ll << 32)) return CYR_UNSUPPORTED;
  // small batches (the single-slot latency path) use 32-parent items so the
  // tree spreads over all SMs; large batches use kTreeThreads-parent items
  long long big_items = 0;
  for (long long t = 0, q = 1; t < M; ++t, q *= R) big_items += (q + kTreeThreads - 1) / kTreeThreads;
  p.np_item = (big_items * S < 2ll * sm_count) ? 32 : kTreeThreads;
  static const int np_env = [] {  // CYR_TREE_NP: parents per work item, 32/64/128 (A/B)
    const char* e = getenv("CYR_TREE_NP");
    return e ? atoi(e) : 0;
  }();
  if (np_env == 32 || np_env == 64 || np_env == 128) p.np_item = np_env;
  long long parents = 1, nodes = 0;
  p.level_blocks[0] = 0;
  for (int t = 0; t < M; ++t) {
    p.level_parents[t] = parents;
    p.child_off[t] = nodes;
    const long long blocks = (parents + p.np_item - 1) / p.np_item;
    p.level_blocks[t + 1] = p.level_blocks[t] + (int)blocks;
    nodes += parents * R;
    parents *= R;
  }
  p.nodes_per_slot = nodes;
  p.blocks_per_slot = p.level_blocks[M];
  if ((long long)S * p.blocks_per_slot >= (1ll << 31)) return CYR_UNSUPPORTED;
  return CYR_OK;
}

}  // namespace cyr

int cyr_launch_tree(const int32_t* codebook, int S, int E, int cap, int M, int16_t* out,
                    int sm_count, cudaStream_t stream) {
  if (S <= 0) return CYR_OK;
  cyr::TreeParams p{};
  const int rc = cyr::tree_params(p, codebook, S, E, cap, M, out, sm_count);
  if (rc != CYR_OK) return rc;
  return cyr::launch_tree_ch<false>(p, sm_count, stream);
}

int cyr_launch_tree_score(const int32_t* codebook, const int32_t* alloc, const double* margin,
                          const double* prob, int S, int E, int cap, int M, int N, int16_t* out,
                          uint32_t* leaf_ok, double* expect, int sm_count, cudaStream_t stream) {
  if (S <= 0) return CYR_OK;
  if (N <= 0 || N > 32767) return CYR_BAD_ARG;
  cyr::TreeParams p{};
  int rc = cyr::tree_params(p, codebook, S, E, cap, M, out, sm_count);
  if (rc != CYR_OK) return rc;
  p.alloc = alloc;
  p.margin = margin;
  p.prob = prob;
  p.N = N;
  p.leaf_ok = leaf_ok;
  const int items = p.level_blocks[M] - p.level_blocks[M - 1];
  double* partial = nullptr;
  if (cyr::malloc_async(reinterpret_cast<void**>(&partial), (size_t)S * items * 2 * sizeof(double),
                      stream) != cudaSuccess)
    return CYR_CUDA_ERROR;
  p.partial = partial;
  rc = cyr::launch_tree_ch<true>(p, sm_count, stream);
  if (rc == CYR_OK && expect != nullptr) {
    cyr::tree_score_reduce_kernel<<<(S + 127) / 128, 128, 0, stream>>>(partial, items, S, N, expect);
    if (cudaPeekAtLastError() != cudaSuccess) rc = CYR_CUDA_ERROR;
  }
  cudaFreeAsync(partial, stream);
  return rc;
}

// ------------------------------------------------ leaf scoring from states
// Mode-T trees (no codebook columns: every node has its own decision) are
// scored from the leaf records themselves: for leaves [first, first + count)
// of level M of each slot (a subtree shard's leaves are one contiguous run),
// the threshold decoder of every user (phy.py:73-80 via decode_user,
// phy.py:196-198), lost / goodput SCs (core.py:132-153) and the leaf weight
// prod_tau prob[tau][k_tau] (digits of the leaf's level-M index, first
// mini-slot most significant).  Per 256-leaf block a fixed-order shared
// reduction, then the blocks in order: deterministic.  This is the per-leaf
// SUMMARY a subtree shard ships instead of its node records.
namespace cyr {
constexpr int kLeafThreads = 256;

__global__ void __launch_bounds__(kLeafThreads) leaf_states_score_kernel(
    const int16_t* __restrict__ leaves, long long slot_stride, int E, int epad, long long first,
    long long count, int R, int M, const int32_t* __restrict__ alloc,
    const double* __restrict__ margin, const double* __restrict__ prob, uint32_t* __restrict__ ok,
    double* __restrict__ partial, int blocks_per_slot) {
  __shared__ double s_lost[kLeafThreads], s_good[kLeafThreads];
  const int s = blockIdx.x / blocks_per_slot, blk = blockIdx.x % blocks_per_slot;
  const long long i = (long long)blk * kLeafThreads + threadIdx.x;
  double lost_w = 0.0, good_w = 0.0;
  if (i < count) {
    const int16_t* rec = leaves + s * slot_stride + i * epad;
    long long total = 0, lost = 0;
    double w = 1.0;
    unsigned q = (unsigned)(first + i);  // leaves < 2^31 (checked by the launcher)
    for (int tau = M - 1; tau >= 0; --tau) {  // last digit = last mini-slot
      const unsigned qd = q / (unsigned)R;
      w *= prob[tau * R + (int)(q - qd * (unsigned)R)];
      q = qd;
    }
    uint32_t bits = 0;
    for (int e = 0; e < E; ++e) {
      const int n = alloc[(long long)s * E + e];
      const double budget = margin[(long long)s * E + e] * (double)(M * n);
      const bool good = n <= 0 || (double)rec[e] <= budget;
      bits |= good ? 1u << e : 0u;
      if (n > 0) {
        total += n;
        if (!good) lost += n;
      }
    }
    if (ok) ok[s * count + i] = bits;
    lost_w = w * (double)lost;
    good_w = w * (double)(total - lost);
  }
  s_lost[threadIdx.x] = lost_w;
  s_good[threadIdx.x] = good_w;
  __syncthreads();
  for (int h = kLeafThreads / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      s_lost[threadIdx.x] += s_lost[threadIdx.x + h];
      s_good[threadIdx.x] += s_good[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[((long long)s * blocks_per_slot + blk) * 2] = s_lost[0];
    partial[((long long)s * blocks_per_slot + blk) * 2 + 1] = s_good[0];
  }
}
// per slot: the blocks' partials in a fixed order (thread t sums blocks
// t, t + 256, ...; then a fixed shared-memory tree): deterministic
__global__ void __launch_bounds__(kLeafThreads) leaf_partials_reduce_kernel(
    const double* __restrict__ partial, int blocks_per_slot, int N, double* __restrict__ expect) {
  __shared__ double s_lost[kLeafThreads], s_good[kLeafThreads];
  const int s = blockIdx.x;
  double l = 0.0, g = 0.0;
  for (int b = threadIdx.x; b < blocks_per_slot; b += kLeafThreads) {
    l += partial[((long long)s * blocks_per_slot + b) * 2];
    g += partial[((long long)s * blocks_per_slot + b) * 2 + 1];
  }
  s_lost[threadIdx.x] = l;
  s_good[threadIdx.x] = g;
  __syncthreads();
  for (int h = kLeafThreads / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      s_lost[threadIdx.x] += s_lost[threadIdx.x + h];
      s_good[threadIdx.x] += s_good[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    expect[s * 3] = -s_lost[0] / (double)N;  // E[r] (core.py:132-146)
    expect[s * 3 + 1] = s_good[0];           // E[goodput SCs] (core.py:149-153)
    expect[s * 3 + 2] = s_lost[0];           // E[lost SCs]
  }
}
}  // namespace cyr

int cyr_launch_leaf_states_score(const int16_t* leaves, long long slot_stride, int S, int E,
                                 int epad, long long first, long long count, int cap, int M,
                                 const int32_t* alloc, const double* margin, const double* prob,
                                 int N, uint32_t* ok, double* expect, cudaStream_t stream) {
  if (S <= 0 || count <= 0) return CYR_OK;
  const long long bps = (count + cyr::kLeafThreads - 1) / cyr::kLeafThreads;
  if (bps * S >= (1ll << 31) || first + count >= (1ll << 31)) return CYR_UNSUPPORTED;
  double* partial = nullptr;
  if (cyr::malloc_async(reinterpret_cast<void**>(&partial), (size_t)S * bps * 2 * sizeof(double),
                      stream) != cudaSuccess)
    return CYR_CUDA_ERROR;
  cyr::leaf_states_score_kernel<<<(unsigned)(bps * S), cyr::kLeafThreads, 0, stream>>>(
      leaves, slot_stride, E, epad, first, count, cap + 1, M, alloc, margin, prob, ok, partial,
      (int)bps);
  cyr::leaf_partials_reduce_kernel<<<S, cyr::kLeafThreads, 0, stream>>>(partial, (int)bps, N,
                                                                         expect);
  cudaFreeAsync(partial, stream);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}
