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
// A node record is the per-user cumulative puncture count as int16, padded to
// Epad = roundup(E, 8) lanes (16/32/48/64 bytes): 128-bit vector granules.
//
// B200 design (HBM-write-bound): a persistent grid walks work items =
// (slot, level, block of NP parents).  Codebook column 0 is the all-zero
// vector (engine.py:112), so leading zero digits add nothing and a parent's
// state is T3[p mod R^3] + T3[p div R^3] (+ T3[...] for deeper trees) where
// T3 holds the sums of every 3-digit suffix — two shared-memory lookups
// instead of a per-digit divide-and-add loop.  The cap+1 codebook columns
// live in registers; each child is one packed 16-bit vector add per
// 16-byte granule into a shared-memory staging buffer, and one thread then
// writes the whole contiguous child run with a single TMA bulk store
// (cp.async.bulk.global.shared::cta, SASS UBLKCP).  Two staging buffers let
// the next item's compute overlap the previous item's store.  A codebook
// whose column 0 is not zero falls back to the per-digit sum.
#include "cyrus_internal.cuh"
#include "cyrus_b200.h"

#include <algorithm>

namespace cyr {

constexpr int kTreeThreads = 256;  // max parents per work item (= threads per CTA)
constexpr int kMaxLevels = 16;

struct TreeParams {
  const int32_t* codebook;
  int16_t* out;
  int S, E, cap, M, epad;
  int np_item;                       // parents per work item (= blockDim.x)
  int r3;                            // (cap+1)^3
  unsigned r3_magic;                 // floor(q / r3) == __umulhi(q, r3_magic) in range
  long long nodes_per_slot;
  int blocks_per_slot;
  int level_blocks[kMaxLevels + 1];  // prefix over parent levels t = 0..M-1
  long long level_parents[kMaxLevels];
  long long child_off[kMaxLevels];   // node offset of level t+1 within a slot
};

__device__ __forceinline__ uint4 vadd16(uint4 a, uint4 b) {
  return make_uint4(__vadd2(a.x, b.x), __vadd2(a.y, b.y), __vadd2(a.z, b.z), __vadd2(a.w, b.w));
}

template <int CH, int R>  // CH: 16-byte granules per record; R = cap + 1
__global__ void __launch_bounds__(kTreeThreads, 2) tree_kernel(const TreeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int NP = p.np_item;
  const size_t stage_bytes = (size_t)NP * R * CH * 16;
  const int r3 = p.r3;
  uint4* t3 = reinterpret_cast<uint4*>(smem + 2 * stage_bytes);  // [r3][CH], per item
  int16_t* bookw = reinterpret_cast<int16_t*>(t3 + (size_t)r3 * CH);  // [R][CH*8]
  const int tid = threadIdx.x;
  const int items = p.S * p.blocks_per_slot;  // host-checked to fit in int
  int it = 0;
  for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
    const int buf = it & 1;
    uint4* stage = reinterpret_cast<uint4*>(smem + buf * stage_bytes);
    const int s = w / p.blocks_per_slot;
    const int bw = w - s * p.blocks_per_slot;
    int t = 0;
    while (bw >= p.level_blocks[t + 1]) ++t;
    const int p0 = (bw - p.level_blocks[t]) * NP;
    const int np = (int)min((long long)NP, p.level_parents[t] - p0);

    if (tid == 0) bulk_wait_read<1>();  // the store issued two items ago released this stage
    // this slot's codebook as packed int16 granules: cooperative load to
    // shared memory, then every thread keeps the cap+1 columns in registers
    const int32_t* cb = p.codebook + (long long)s * R * p.E;
    for (int idx = tid; idx < R * CH * 8; idx += NP) {
      const int k = idx / (CH * 8), e = idx % (CH * 8);
      bookw[idx] = (int16_t)((e < p.E) ? cb[k * p.E + e] : 0);
    }
    __syncthreads();
    uint4 col[R][CH];
#pragma unroll
    for (int k = 0; k < R; ++k)
#pragma unroll
      for (int c = 0; c < CH; ++c) col[k][c] = reinterpret_cast<const uint4*>(bookw)[k * CH + c];
    const uint4 c0 = col[0][0];
    bool zero0 = (c0.x | c0.y | c0.z | c0.w) == 0u;
#pragma unroll
    for (int c = 1; c < CH; ++c)
      zero0 = zero0 && (col[0][c].x | col[0][c].y | col[0][c].z | col[0][c].w) == 0u;

    // suffix table (also reused across items: rebuilt per item, it is small)
    for (int x = tid; x < r3; x += NP) {
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
      uint4* dst = stage + (size_t)tid * R * CH;
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int c = 0; c < CH; ++c) dst[k * CH + c] = vadd16(cum[c], col[k][c]);
    }
    fence_proxy_async_smem();  // generic smem writes -> visible to the bulk-copy proxy
    __syncthreads();
    if (tid == 0) {
      const long long first = (long long)s * p.nodes_per_slot + p.child_off[t] + (long long)p0 * R;
      bulk_s2g(p.out + first * p.epad, stage, (uint32_t)((size_t)np * R * CH * 16));
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_all();
}

template <int CH, int R>
int launch_tree_t(const TreeParams& p, int sm_count, cudaStream_t stream) {
  const size_t smem =
      2 * (size_t)p.np_item * R * CH * 16 + (size_t)p.r3 * CH * 16 + (size_t)R * CH * 16;
  if (smem > 227 * 1024) return CYR_UNSUPPORTED;
  if (cudaFuncSetAttribute(tree_kernel<CH, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return CYR_CUDA_ERROR;
  const long long items = (long long)p.S * p.blocks_per_slot;
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (227 * 1024) / (smem + 1024)));
  const long long grid = std::min<long long>(items, (long long)sm_count * per_sm);
  tree_kernel<CH, R><<<(unsigned)grid, p.np_item, smem, stream>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

template <int CH>
int launch_tree_r(const TreeParams& p, int sm_count, cudaStream_t stream) {
  switch (p.cap + 1) {
    case 2: return launch_tree_t<CH, 2>(p, sm_count, stream);
    case 3: return launch_tree_t<CH, 3>(p, sm_count, stream);
    case 4: return launch_tree_t<CH, 4>(p, sm_count, stream);
    case 5: return launch_tree_t<CH, 5>(p, sm_count, stream);
    case 6: return launch_tree_t<CH, 6>(p, sm_count, stream);
    case 7: return launch_tree_t<CH, 7>(p, sm_count, stream);
    case 8: return launch_tree_t<CH, 8>(p, sm_count, stream);
    case 9: return launch_tree_t<CH, 9>(p, sm_count, stream);
    default: return CYR_UNSUPPORTED;
  }
}

}  // namespace cyr

int cyr_launch_tree(const int32_t* codebook, int S, int E, int cap, int M, int16_t* out,
                    int sm_count, cudaStream_t stream) {
  if (S <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers || cap < 1 || M < 1 || M > 10) return CYR_BAD_ARG;
  if (cap + 1 > 9) return CYR_UNSUPPORTED;
  cyr::TreeParams p{};
  p.codebook = codebook;
  p.out = out;
  p.S = S;
  p.E = E;
  p.cap = cap;
  p.M = M;
  p.epad = (E + 7) / 8 * 8;
  const long long R = cap + 1;
  p.r3 = (int)(R * R * R);
  // ceil(2^32 / r3): floor(q * magic / 2^32) == floor(q / r3) while
  // q * (magic * r3 - 2^32) < 2^32, i.e. for every q < 2^32 / r3
  p.r3_magic = (unsigned)((0x100000000ull + p.r3 - 1) / p.r3);
  long long top = 1;
  for (int t = 0; t < M - 1; ++t) top *= R;
  if (top * p.r3 >= (1ll << 32)) return CYR_UNSUPPORTED;
  // small batches (the single-slot latency path) use 64-parent items so the
  // tree spreads over all SMs; large batches use 256-parent items
  long long big_items = 0;
  for (long long t = 0, q = 1; t < M; ++t, q *= R) big_items += (q + 255) / 256;
  p.np_item = (big_items * S < 2ll * sm_count) ? 64 : cyr::kTreeThreads;
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
  switch (p.epad / 8) {
    case 1: return cyr::launch_tree_r<1>(p, sm_count, stream);
    case 2: return cyr::launch_tree_r<2>(p, sm_count, stream);
    case 3: return cyr::launch_tree_r<3>(p, sm_count, stream);
    default: return cyr::launch_tree_r<4>(p, sm_count, stream);
  }
}
