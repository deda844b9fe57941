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
// Epad = roundup(E, 8) lanes (16/32/64 bytes): 128-bit vector granules.
//
// B200 design (HBM-write-bound): a persistent grid (2 CTAs per SM) walks
// work items = (slot, level, block of 256 parents).  Each thread rebuilds its
// parent's record from the parent's base-(cap+1) digits (no parent reads from
// HBM at all), adds every codebook column with packed 16-bit vector adds, and
// drops the (cap+1) children into a shared-memory staging buffer; one thread
// then writes the whole contiguous child run with a single TMA bulk store
// (cp.async.bulk.global.shared::cta, SASS UBLKCP).  Two staging buffers let
// the next item's compute overlap the previous item's store.
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
  long long nodes_per_slot;
  int blocks_per_slot;
  int level_blocks[kMaxLevels + 1];  // prefix over parent levels t = 0..M-1
  long long level_parents[kMaxLevels];
  long long child_off[kMaxLevels];   // node offset of level t+1 within a slot
};

__device__ __forceinline__ uint4 vadd16(uint4 a, uint4 b) {
  return make_uint4(__vadd2(a.x, b.x), __vadd2(a.y, b.y), __vadd2(a.z, b.z), __vadd2(a.w, b.w));
}

template <int CH>  // 16-byte granules per record (Epad / 8)
__global__ void __launch_bounds__(kTreeThreads, 2) tree_kernel(const TreeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int R = p.cap + 1;
  const int NP = p.np_item;
  const size_t stage_bytes = (size_t)NP * R * CH * 16;
  const int tid = threadIdx.x;
  const long long items = (long long)p.S * p.blocks_per_slot;
  int it = 0;
  for (long long w = blockIdx.x; w < items; w += gridDim.x, ++it) {
    const int buf = it & 1;
    uint4* stage = reinterpret_cast<uint4*>(smem + buf * stage_bytes);
    uint4* book = reinterpret_cast<uint4*>(smem + 2 * stage_bytes + (size_t)buf * R * CH * 16);
    const int s = (int)(w / p.blocks_per_slot);
    const int bw = (int)(w % p.blocks_per_slot);
    int t = 0;
    while (bw >= p.level_blocks[t + 1]) ++t;
    const long long p0 = (long long)(bw - p.level_blocks[t]) * NP;
    const int np = (int)min((long long)NP, p.level_parents[t] - p0);

    if (tid == 0) bulk_wait_read<1>();  // the store issued two items ago released stage
    // this slot's codebook as int16 records: book[k][granule]
    for (int idx = tid; idx < R * CH * 8; idx += NP) {
      const int k = idx / (CH * 8), e = idx % (CH * 8);
      const int v = (e < p.E) ? p.codebook[((long long)s * R + k) * p.E + e] : 0;
      reinterpret_cast<int16_t*>(book)[idx] = (int16_t)v;
    }
    __syncthreads();

    if (tid < np) {
      uint4 cum[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) cum[c] = make_uint4(0, 0, 0, 0);
      unsigned q = (unsigned)(p0 + tid);  // < (cap+1)^(M-1) <= 2^31 (host-checked)
      for (int d = 0; d < t; ++d) {
        const unsigned nq = q / (unsigned)R;
        const int k = (int)(q - nq * (unsigned)R);
        q = nq;
#pragma unroll
        for (int c = 0; c < CH; ++c) cum[c] = vadd16(cum[c], book[k * CH + c]);
      }
      uint4* dst = stage + (size_t)tid * R * CH;
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int c = 0; c < CH; ++c) dst[k * CH + c] = vadd16(cum[c], book[k * CH + c]);
    }
    fence_proxy_async_smem();  // generic smem writes -> visible to the bulk-copy proxy
    __syncthreads();
    if (tid == 0) {
      const long long first = (long long)s * p.nodes_per_slot + p.child_off[t] + p0 * R;
      bulk_s2g(p.out + first * p.epad, stage, (uint32_t)((size_t)np * R * CH * 16));
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_all();
}

template <int CH>
int launch_tree_t(const TreeParams& p, int sm_count, cudaStream_t stream) {
  const int R = p.cap + 1;
  const size_t smem = 2 * (size_t)p.np_item * R * CH * 16 + 2 * (size_t)R * CH * 16;
  if (smem > 227 * 1024) return CYR_UNSUPPORTED;
  if (cudaFuncSetAttribute(tree_kernel<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return CYR_CUDA_ERROR;
  const long long items = (long long)p.S * p.blocks_per_slot;
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (227 * 1024) / (smem + 1024)));
  const long long grid = std::min<long long>(items, (long long)sm_count * per_sm);
  tree_kernel<CH><<<(unsigned)grid, p.np_item, smem, stream>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

}  // namespace cyr

int cyr_launch_tree(const int32_t* codebook, int S, int E, int cap, int M, int16_t* out,
                    int sm_count, cudaStream_t stream) {
  if (S <= 0) return CYR_OK;
  if (E < 1 || E > cyr::kMaxUsers || cap < 1 || M < 1 || M > cyr::kMaxLevels) return CYR_BAD_ARG;
  cyr::TreeParams p{};
  p.codebook = codebook;
  p.out = out;
  p.S = S;
  p.E = E;
  p.cap = cap;
  p.M = M;
  p.epad = (E + 7) / 8 * 8;
  const long long R = cap + 1;
  long long top = 1;
  for (int t = 0; t < M - 1; ++t) top *= R;
  if (top > (1ll << 31)) return CYR_UNSUPPORTED;  // parent indices are 32-bit
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
    if (p.level_blocks[t] + blocks > (1ll << 30)) return CYR_UNSUPPORTED;
    p.level_blocks[t + 1] = p.level_blocks[t] + (int)blocks;
    nodes += parents * R;
    parents *= R;
  }
  p.nodes_per_slot = nodes;
  p.blocks_per_slot = p.level_blocks[M];
  switch (p.epad / 8) {
    case 1: return cyr::launch_tree_t<1>(p, sm_count, stream);
    case 2: return cyr::launch_tree_t<2>(p, sm_count, stream);
    case 3: return cyr::launch_tree_t<3>(p, sm_count, stream);
    default: return cyr::launch_tree_t<4>(p, sm_count, stream);
  }
}
