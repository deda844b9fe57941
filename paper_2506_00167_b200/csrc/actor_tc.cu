// actor_tc.cu — K2-TC: the actor MLP on the 5th-generation tensor cores.
//
// Optional bf16 path (precision CYR_BF16_TC) for batches where the MLP is a
// real dense GEMM — Mode-T tree levels and large Mode-R batches (SURVEY.md
// §7 step 8, BASELINE configs[4]).  Decisions are not bit-comparable with
// the fp32/fp64 paths (bf16 operands); tests report the agreement rate.
//
// One CTA (4 warps) owns M = 128 batch columns and runs every layer:
//   D[128 x N] (fp32, TMEM) = A[128 x K] (bf16, smem) . W[N x K]^T (bf16, smem)
// with tcgen05.mma.cta_group::1.kind::f16 issued by one thread, 16-deep K
// steps.  Both operands are K-major SWIZZLE_128B tiles of 64 K-elements:
//   * W tiles are pre-swizzled at publish time into exactly that smem image
//     (cyr_policy_create), so one TMA bulk copy (cp.async.bulk, UBLKCP) per
//     tile lands them MMA-ready; a 3-slot ring streams them across layers,
//     slots released by tcgen05.commit on an mbarrier;
//   * A is the activation tile: layer 1 is built from the branch / node-state
//     features, later layers are written by the previous layer's epilogue
//     (tcgen05.ld 32x32b -> bias, ReLU -> bf16 -> swizzled st.shared).
// The last layer's epilogue writes fp32 logits raw[col][2E] for K3.
// Widths <= 256 (N of one MMA, 256 TMEM columns); wider actors use SIMT.
#include "cyrus_internal.cuh"
#include "actor_common.cuh"
#include "cyrus_b200.h"

#include <cuda_bf16.h>
#include <cstdio>

namespace cyr {

constexpr int kTcThreads = 128;
constexpr int kTcM = 128;
constexpr int kTcSlots = 3;
constexpr int kTcSlotBytes = 256 * 128;  // one [256 x 64] bf16 tile
constexpr int kTcMaxKt = 4;              // K <= 256

struct TcLaunch {
  ActorDesc desc;
  const unsigned char* tc_blob;  // per layer: Kt tiles of [npad x 64] bf16, SW128 images
  long long tc_off[kMaxLayers];  // byte offset of layer l's first tile
  int tc_npad[kMaxLayers];       // N padded to a multiple of 16
  const float* bias;             // fp32 bias per layer at desc.layer[l].b_off (fp32 blob)
  const int32_t* alloc;
  float* raw;
  int S, E, N, cap, ncols;
  // Mode T
  int mode_t;
  const int16_t* node;
  const int32_t* mcs;
  long long nodes_per_slot, parent_off;
  int parent_base;  // level index of the first parent (subtree shards)
  int parents, tau, M, epad;
  double mcs_scale;
};

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);  // start address (16-B units)
  d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;             // SBO: 8-row core-matrix groups
  d |= (uint64_t)1 << 46;                       // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

// byte offset of element (row r, k in [0,64)) in a K-major SW128 bf16 tile
__host__ __device__ __forceinline__ uint32_t sw128_offset(int r, int k) {
  const int chunk = (k * 2) >> 4;  // 16-byte chunk within the 128-byte row
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((chunk ^ (r & 7)) << 4) + ((k * 2) & 15));
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// MMA issue is warp-wide: the WHOLE (converged) warp runs the issue loop and
// elect.sync inside each asm picks the one lane that issues.  Issued from
// inside `if (lane == 0)`, ptxas cannot prove the operands uniform and wraps
// every tcgen05.mma / commit in an ELECT + R2UR.BROADCAST + BRA.U.ANY
// waterfall (~146 cycles per instruction whatever N).
__device__ __forceinline__ void tc_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
// Four consecutive K steps (K = 64, one SW128 K tile) in ONE asm statement,
// the per-step operands derived INSIDE the asm from one base each.  Measured
// (scripts/micro/mma_rate.cu, M = 128, TS): one asm per MMA 146 cycles per
// instruction whatever N; four per asm with the operands precomputed in C
// (each a separate R2UR) 52-59; four per asm with in-asm adds 17.5 for
// N = 32, 33 for N = 64, 129 for N = 256 -- the tensor-pipe floor
// 128 * N / 256.  B descriptors of consecutive K steps inside one SW128 atom
// are 32 bytes (+2 in the start-address field) apart; A columns in TMEM 8.
__device__ __forceinline__ void tc_mma_ts_x4(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, int accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 ta;\n\t.reg .b64 bd;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "add.u32 ta, %1, 8;\n\tadd.u64 bd, %2, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
      "add.u32 ta, %1, 16;\n\tadd.u64 bd, %2, 4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
      "add.u32 ta, %1, 24;\n\tadd.u64 bd, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_ss_x4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, int accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 ad, bd;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "add.u64 ad, %1, 2;\n\tadd.u64 bd, %2, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %3, 1;\n\t"
      "add.u64 ad, %1, 4;\n\tadd.u64 bd, %2, 4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %3, 1;\n\t"
      "add.u64 ad, %1, 6;\n\tadd.u64 bd, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %3, 1;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}



// K tile t of the layer-1 A operand for batch column `col`, written as row
// `row` of the SW128 image `a` (zeros past in0).  Feature i of the actor
// input, rounded to bf16 from the fp32 value x * (1 / scale) (this path is
// bf16 end to end; fp32 feature math keeps the builders off the fp64
// division sequences):
//   Mode R: [n/N (E), j/cap]
//   Mode T: [n/N (E), k/cap, cum/N (E), mcs/mcs_scale (E), arrivals/(M*cap),
//            (tau-1)/M]
// E = 4 / 10 / 16 take tc_feature_row below (registers, 16-byte stores).
// The generic path decodes the column's indices once, issues every global
// load first (the values parked in local memory) and then stores the bf16
// values by shared-memory address without a "memory" clobber: through the
// generic tile pointer each store was ordered before the next user's loads
// (possible alias), so every batch of loads paid its full latency.
__device__ __forceinline__ void tc_put(uint32_t a, int row, int t, int i, float x) {
  if (i >= t * 64 && i < t * 64 + 64) {
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(a + sw128_offset(row, i - t * 64)),
                 "h"(*reinterpret_cast<const unsigned short*>(&h)));
  }
}

// x / d for 0 <= x < 2^22 from a float reciprocal and one correction step
// (the quotient is off by at most one there); larger x: integer division.
__device__ __forceinline__ int div_small(int x, int d, float inv) {
  if (x >= (1 << 22)) return x / d;
  const int q = (int)((float)x * inv);
  const int r = x - q * d;
  return r < 0 ? q - 1 : (r >= d ? q + 1 : q);
}

// The feature row of one column for a compile-time user count (cfg1 / cfg2 /
// cfg5: E = 4 / 10 / 16; K tile 0, in <= 64): every load issued up front,
// the 64 bf16 values packed in registers (cvt.rn.bf16x2.f32, the same RN
// rounding as the per-element path) and written as 8 16-byte chunks.  The
// per-element path cost ~6.5k cycles per 128-column Mode-T tile (runtime
// integer divisions, 33 scalar stores with their swizzle arithmetic), more
// than the fused MLP's whole block chain.
template <int kE>
__device__ __forceinline__ void tc_feature_row(const TcLaunch& p, int col, uint32_t a, int row) {
  uint32_t w[32];
  if (col >= p.ncols) {
#pragma unroll
    for (int j = 0; j < 32; ++j) w[j] = 0u;
  } else {
    const int cap = p.cap;
    const int g = div_small(col, cap, 1.0f / (float)cap);
    const int k = col - g * cap + 1;
    const int s = p.mode_t ? div_small(g, p.parents, 1.0f / (float)p.parents) : g;
    const int q = p.mode_t ? g - s * p.parents : 0;
    const int32_t* al = p.alloc + (long long)s * kE;
    int av[kE], mv[kE], nv[kE];
#pragma unroll
    for (int e = 0; e < kE; ++e) av[e] = __ldg(al + e);
    float arr = 0.f, tauf = 0.f;
    if (p.mode_t) {
      const int32_t* mc = p.mcs + (long long)s * kE;
      const int16_t* nd =
          p.parent_off >= 0
              ? p.node + ((long long)s * p.nodes_per_slot + p.parent_off + q) * p.epad
              : nullptr;
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        mv[e] = __ldg(mc + e);
        nv[e] = nd ? __ldg(nd + e) : 0;
      }
      int arrivals = 0, x = p.parent_base + q;
      const int base = cap + 1;
      const float inv_base = 1.0f / (float)base;
      for (int d = 1; d < p.tau; ++d) {
        const int xq = div_small(x, base, inv_base);
        arrivals += x - xq * base;
        x = xq;
      }
      arr = (float)arrivals / (float)(p.M * p.cap);
      tauf = (float)(p.tau - 1) / (float)p.M;
    } else {
#pragma unroll
      for (int e = 0; e < kE; ++e) mv[e] = nv[e] = 0;
    }
    const float inv_n = 1.0f / (float)p.N, inv_mcs = (float)(1.0 / p.mcs_scale);
    const float kf = (float)k / (float)p.cap;
    auto feat = [&](int i) -> float {  // i is a compile-time constant after unrolling
      if (i < kE) return (float)av[i] * inv_n;
      if (i == kE) return kf;
      if (!p.mode_t) return 0.f;
      if (i < 2 * kE + 1) return (float)nv[i - kE - 1] * inv_n;
      if (i < 3 * kE + 1) return (float)mv[i - 2 * kE - 1] * inv_mcs;
      if (i == 3 * kE + 1) return arr;
      if (i == 3 * kE + 2) return tauf;
      return 0.f;
    };
#pragma unroll
    for (int j = 0; j < 32; ++j)
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w[j]) : "f"(feat(2 * j + 1)), "f"(feat(2 * j)));
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + sw128_offset(row, c * 8)),
                 "r"(w[4 * c]), "r"(w[4 * c + 1]), "r"(w[4 * c + 2]), "r"(w[4 * c + 3]));
}

__device__ __forceinline__ void tc_feature_tile(const TcLaunch& p, int col, int t,
                                                unsigned char* tile, int row) {
  const uint32_t a = smem_u32(tile);
  if (t == 0 && p.desc.layer[0].in <= 64) {
    switch (p.E) {
      case 4: tc_feature_row<4>(p, col, a, row); return;
      case 10: tc_feature_row<10>(p, col, a, row); return;
      case 16: tc_feature_row<16>(p, col, a, row); return;
      default: break;
    }
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a + sw128_offset(row, c * 8)),
                 "r"(0u));
  if (col >= p.ncols) return;
  const int E = p.E;
  const int k = col % p.cap + 1;
  const int g = col / p.cap;
  const int s = p.mode_t ? g / p.parents : g;
  const int q = p.mode_t ? g - s * p.parents : 0;
  const int32_t* al = p.alloc + (long long)s * E;
  const int32_t* mc = p.mode_t ? p.mcs + (long long)s * E : nullptr;
  const int16_t* nd =
      (p.mode_t && p.parent_off >= 0)
          ? p.node + ((long long)s * p.nodes_per_slot + p.parent_off + q) * p.epad
          : nullptr;
  const float inv_n = 1.0f / (float)p.N, inv_mcs = (float)(1.0 / p.mcs_scale);
  // every global load first (one latency for the column, not one per batch
  // of users), the values parked in local memory (L1), then the stores
  int v[3 * kMaxUsers];
  for (int e = 0; e < E; ++e) {
    v[e] = __ldg(al + e);
    if (p.mode_t) {
      v[kMaxUsers + e] = nd ? __ldg(nd + e) : 0;
      v[2 * kMaxUsers + e] = __ldg(mc + e);
    }
  }
  for (int e = 0; e < E; ++e) {
    tc_put(a, row, t, e, (float)v[e] * inv_n);
    if (p.mode_t) {
      tc_put(a, row, t, E + 1 + e, (float)v[kMaxUsers + e] * inv_n);
      tc_put(a, row, t, 2 * E + 1 + e, (float)v[2 * kMaxUsers + e] * inv_mcs);
    }
  }
  tc_put(a, row, t, E, (float)k / (float)p.cap);
  if (p.mode_t) {
    int arrivals = 0, x = p.parent_base + q;
    for (int d = 1; d < p.tau; ++d) {
      arrivals += x % (p.cap + 1);
      x /= (p.cap + 1);
    }
    tc_put(a, row, t, 3 * E + 1, (float)arrivals / (float)(p.M * p.cap));
    tc_put(a, row, t, 3 * E + 2, (float)(p.tau - 1) / (float)p.M);
  }
}

__global__ void __launch_bounds__(kTcThreads, 1) actor_tc_kernel(const TcLaunch p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B aligned carve-up: A tiles | B ring | barriers
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* a_tiles = base;                                   // kTcMaxKt x 16 KB
  unsigned char* ring = base + kTcMaxKt * kTcM * 128;              // kTcSlots x 32 KB
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(ring + kTcSlots * kTcSlotBytes);
  uint64_t* bar_free = bar_full + kTcSlots;
  uint64_t* bar_mma = bar_free + kTcSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_mma + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int c0 = blockIdx.x * kTcM;
  const int nl = p.desc.n_layers;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kTcSlots; ++i) {
      mbar_init(&bar_full[i], 1);
      mbar_init(&bar_free[i], 1);
    }
    mbar_init(bar_mma, 1);
    fence_mbar_init();
  }

  // weight-tile sequence across layers: g -> (layer, k-tile)
  int total = 0;
  for (int l = 0; l < nl; ++l) total += (p.desc.layer[l].in + 63) / 64;
  auto tile_of = [&](int g, int& l, int& t) {
    l = 0;
    int first = 0;
    for (;; ++l) {
      const int kt = (p.desc.layer[l].in + 63) / 64;
      if (g < first + kt) break;
      first += kt;
    }
    t = g - first;
  };
  auto issue = [&](int g) {  // thread 0
    if (g >= total) return;
    const int slot = g % kTcSlots;
    if (g >= kTcSlots) mbar_wait(&bar_free[slot], (uint32_t)(((g / kTcSlots) - 1) & 1));
    int l, t;
    tile_of(g, l, t);
    const uint32_t bytes = (uint32_t)p.tc_npad[l] * 128;
    mbar_expect_tx(&bar_full[slot], bytes);
    bulk_g2s(ring + (size_t)slot * kTcSlotBytes, p.tc_blob + p.tc_off[l] + (long long)t * bytes,
             bytes, &bar_full[slot]);
  };

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0)
    for (int g = 0; g < kTcSlots - 1; ++g) issue(g);

  // layer-1 A tile(s): thread tid builds batch column c0 + tid
  {
    const int kt0 = (p.desc.layer[0].in + 63) / 64;
    for (int t = 0; t < kt0; ++t) tc_feature_tile(p, c0 + tid, t, a_tiles + t * kTcM * 128, tid);
  }
  fence_proxy_async_smem();
  __syncthreads();

  int g = 0, mma_phase = 0;
  for (int l = 0; l < nl; ++l) {
    const LayerDesc& L = p.desc.layer[l];
    const int kt = (L.in + 63) / 64;
    const int npad = p.tc_npad[l];
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(npad >> 3) << 17) |
                           ((uint32_t)(kTcM >> 4) << 24);
    if (warp == 0) {  // whole warp: the K-tile asm elects the issuing lane
      tc_fence_after();
      for (int t = 0; t < kt; ++t, ++g) {
        const int slot = g % kTcSlots;
        mbar_wait(&bar_full[slot], (uint32_t)((g / kTcSlots) & 1));
        tc_fence_after();
        const uint32_t a_addr = smem_u32(a_tiles + t * kTcM * 128);
        const uint32_t b_addr = smem_u32(ring + (size_t)slot * kTcSlotBytes);
        tc_mma_ss_x4(tmem, umma_desc_sw128(a_addr), umma_desc_sw128(b_addr), idesc, t > 0 ? 1 : 0);
        tc_commit_w(&bar_free[slot]);  // slot reusable once these MMAs retire
        if (lane == 0) issue(g + kTcSlots - 1);  // refill the slot freed by the previous tile
        __syncwarp();
      }
      tc_commit_w(bar_mma);  // accumulator complete
    }
    // epilogue: TMEM lane (32*warp + lane) = batch column c0 + tid
    mbar_wait(bar_mma, (uint32_t)(mma_phase & 1));
    ++mma_phase;
    tc_fence_after();
    const bool last = l == nl - 1;
    const int col = c0 + tid;
    const float* bias = p.bias + L.b_off;
    // hidden layers also zero the K padding of the next A tile (n0 < roundup(out, 64))
    const int n_end = last ? npad : ((L.out + 63) & ~63);
    for (int n0 = 0; n0 < n_end; n0 += 32) {
      uint32_t r[32];
      if (n0 < npad) tc_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)n0, r);
      else
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      if (last) {
        if (col < p.ncols)
          for (int j = 0; j < 32; ++j) {
            const int o = n0 + j;
            if (o < L.out) p.raw[(long long)col * L.out + o] = __uint_as_float(r[j]) + bias[o];
          }
      } else {
        unsigned char* a = a_tiles + (n0 >> 6) * kTcM * 128;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int o = n0 + j;
          float v0 = o < L.out ? __uint_as_float(r[j]) + bias[o] : 0.f;
          float v1 = o + 1 < L.out ? __uint_as_float(r[j + 1]) + bias[o + 1] : 0.f;
          v0 = v0 > 0.f ? v0 : 0.f;
          v1 = v1 > 0.f ? v1 : 0.f;
          *reinterpret_cast<__nv_bfloat162*>(a + sw128_offset(tid, (n0 & 63) + j)) =
              __floats2bfloat162_rn(v0, v1);
        }
      }
    }
    fence_proxy_async_smem();  // new A tiles -> visible to the MMA (async proxy)
    tc_fence_before();
    __syncthreads();
  }
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

// ------------------------------------------------------------ fused narrow
// Narrow 3-layer actors (Mode T cfg1/cfg2: [3E+3, <=256, <=256, 2E]) on big
// levels: ONE persistent kernel, one CTA per SM, every weight resident in
// shared memory for the whole launch (W1 32 KB + W2 128 KB + W3 16 KB at
// cfg2, loaded once by TMA), and the hidden activations never leave the SM:
//
//   features (smem, SW128)  --MMA1-->  D1 (TMEM, fp32)  --epi1-->  A2 (TMEM, bf16)
//   A2 (TMEM)               --MMA2-->  D2 (TMEM)        --epi2-->  A3 (TMEM, bf16)
//   A3 (TMEM)               --MMA3-->  D3 (TMEM)        --epi3-->  raw logits (HBM)
//
// MMA2 / MMA3 read their A operand straight from tensor memory
// (tcgen05.mma ... [d], [a_tmem], b_desc: lane = batch column, column c =
// K elements 2c, 2c+1), so the layer-by-layer path's 3 x 1 GB of HBM
// activation images at the deepest cfg2 level become on-chip traffic.
// TMEM (512 columns): D1 / D2 at [0, 256), A2 at [256, 384), A3 at [384, 512),
// D3 at [256, 256 + N3) (A2 is dead once MMA2 has completed).
// Roles:
//   warps 0-15  epilogues: warp w reads TMEM lane quarter w % 4; per layer it
//               converts a chunk of N half 0 (columns part * n/8 of it, part
//               = w / 4), arrives, then the same chunk of half 1 (packed bias
//               add, ReLU folded into the bf16x2 convert, tcgen05.st); after
//               MMA3 each warp reads 8 head logits (the head epilogue);
//   warps 16-19 feature builders (kFusedGroups groups of 4 warps, group g
//               building the blocks i = g (mod groups) into A1 tile g);
//   last warp   the weight TMA (lane 0) and every MMA (one elected lane).
// A second block in flight would need a second 256-column fp32 accumulator:
// TMEM (512 columns) holds D + A2 + A3 of one block and no more, so the
// overlap comes from splitting each block's chain in N halves instead.
// Measured (scripts/fused_probe.py, 2M Mode-R columns, event timing): 350 us
// = 63 % of the bf16 peak (852 us / 27 % before these changes; 8M columns
// 1,230-1,345 us = 65-71 %); the deepest cfg2 Mode-T level (2M columns,
// 316 GFLOP) 358 us under ncu = 63 %:
//  * MMA issue: the whole warp runs the loop and one asm issues a K tile (4
//    MMAs) under one elect.sync with the per-step operands added inside the
//    asm.  Issued one per asm from inside `lane == 0`, every tcgen05.mma cost
//    ~146 cycles whatever N (ptxas's ELECT / R2UR.BROADCAST / BRA.U.ANY
//    waterfall; scripts/micro/mma_rate.cu); now 17.5 for N = 32, 129 for
//    N = 256 (the pipe floor is 128 * N / 256);
//  * the block chain runs in N halves: MMA1 in two halves, each epilogue in
//    two column chunks per warp (half 0 first, its own barrier), MMA2 half 0
//    over K half 0 as soon as epi1 chunk 0 is in, MMA2 half 1 while epi2
//    chunk 0 runs, MMA3 K half 0 while epi2 chunk 1 runs;
//  * the head output: each epilogue warp reads 8 of D3's columns into
//    registers right after MMA3 and writes them, with the bias, into a
//    row-major shared-memory stage during the next block's MMA2; one bulk
//    copy per block (128 x out fp32 = the block's contiguous slice of raw).
//    As 20 scattered generic 4-byte stores per thread it cost ~3.6k cycles;
//  * feature rows (builders) for E = 4 / 10 / 16 built in registers and
//    written as 8 16-byte chunks; the per-element path (runtime integer
//    divisions, scalar stores through a generic pointer that serialised the
//    next loads) took 6.5k cycles per Mode-T tile, more than the chain;
//  * bias pairs by explicit ld.shared (as generic 64-bit loads they were the
//    kernel's most expensive instructions).
// Per block (CYR_FUSED_PROF trace, CTA 0, 2M Mode-R columns): ~5.2k cycles,
// the tensor pipe busy ~2.9k of them.  A/B knobs (compile-time):
// CYR_FUSED_GROUPS (2 builder groups: Mode R 73.7 % vs 65.3 % at 8M
// columns, Mode T 370 vs 358 us: 1 kept), CYR_FUSED_SPIN (test_wait spinning
// on the hand-off barriers: slower).
#ifndef CYR_FUSED_SPIN
#define CYR_FUSED_SPIN 0
#endif
#if CYR_FUSED_SPIN
#define CYR_FUSED_WAIT mbar_wait_spin
#else
#define CYR_FUSED_WAIT mbar_wait
#endif
#ifndef CYR_FUSED_GROUPS
#define CYR_FUSED_GROUPS 1
#endif
#ifndef CYR_FUSED_EPI
#define CYR_FUSED_EPI 16
#endif
constexpr int kFusedGroups = CYR_FUSED_GROUPS;     // feature-builder groups of 4 warps
constexpr int kFusedEpi = CYR_FUSED_EPI;           // epilogue warps (8 or 16)
constexpr int kFusedParts = kFusedEpi / 4;         // column parts per TMEM lane quarter
static_assert(kFusedEpi == 16, "epilogue chunks are n/8 columns: 4 parts per lane quarter");
constexpr int kFusedMmaWarp = kFusedEpi + 4 * kFusedGroups;
constexpr int kFusedThreads = 32 * (kFusedMmaWarp + 1);
constexpr int kFusedA2Col = 256, kFusedA3Col = 384, kFusedD3Col = 256;

__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

#ifdef CYR_FUSED_PROF
__device__ int g_fused_trace_launch = 0;
#endif
__device__ __forceinline__ void tc_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}

struct FusedLayout {  // shared-memory carve-up (bytes from the 1024-aligned base)
  uint32_t w_off[3], w_bytes[3], feat, bias, bars, stage, stage_bytes, total;
};
constexpr uint32_t kSmemOptinSm100 = 232448;  // 227 KB opt-in per CTA on sm_100

__host__ __device__ inline FusedLayout fused_layout(const ActorDesc& d, const int* npad) {
  FusedLayout f{};
  uint32_t off = 0;
  for (int l = 0; l < 3; ++l) {
    f.w_off[l] = off;
    f.w_bytes[l] = (uint32_t)((d.layer[l].in + 63) / 64) * (uint32_t)npad[l] * 128u;
    off += (f.w_bytes[l] + 1023u) & ~1023u;
  }
  f.feat = off;
  off += (kFusedGroups < 2 ? 2 : kFusedGroups) * kTcM * 128;
  f.bias = off;
  off += (uint32_t)(npad[0] + npad[1] + npad[2]) * 4u;
  off = (off + 7u) & ~7u;
  f.bars = off;
  off += 32 * 8 + 16;
  // head output stage: the block's [128 x out] fp32 logits, row-major, i.e.
  // exactly its contiguous slice of `raw`, written by one bulk copy instead
  // of 128 threads x out scattered 4-byte stores (80-byte stride: every warp
  // store touched 32 sectors; ~3.6k cycles per block on the critical path).
  // Left out (stage_bytes = 0, direct stores) when it would not fit.
  off = (off + 127u) & ~127u;
  const uint32_t sb = (uint32_t)kTcM * (uint32_t)d.layer[2].out * 4u;
  if (off + sb + 1024 <= kSmemOptinSm100) {
    f.stage = off;
    f.stage_bytes = sb;
    off += sb;
  }
  f.total = off + 1024;  // alignment slack
  return f;
}

// One column chunk of a hidden-layer epilogue: this warp's TMEM lane
// quarter, D columns [c0, c0 + W) (fp32) -> bias, ReLU -> bf16 pairs into A
// columns [a_col + c0 / 2, + W / 2).  Per column pair one packed fp32 add of
// the bias pair (add.rn.f32x2, bit-identical to two FADDs) and one convert
// with the ReLU folded in (cvt.rn.relu.bf16x2.f32: max(x, 0) then round, low
// half = even K).  Waits for its TMEM stores.
template <int W>
__device__ __forceinline__ void fused_epi_chunk(uint32_t tmem, int quarter, int c0, int a_col,
                                                const float* bias) {
  const uint32_t lanes = (uint32_t)(quarter * 32) << 16;
  uint32_t r[W];
  if constexpr (W == 32) tc_ld32(tmem + lanes + (uint32_t)c0, r);
  else tc_ld16(tmem + lanes + (uint32_t)c0, r);
  // bias pairs by ld.shared.v2.b64 (explicit shared state space: through the
  // generic pointer these loads were 19 % of the kernel's instructions' cost)
  const uint32_t bs = smem_u32(bias + c0);
  uint32_t w[W / 2];
#pragma unroll
  for (int j = 0; j < W / 2; j += 2) {
    unsigned long long b01, b23;
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(b01), "=l"(b23) : "r"(bs + 8u * j));
    unsigned long long v0, v1;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(v0) : "l"(f32x2_pack(__uint_as_float(r[2 * j]),
                                                              __uint_as_float(r[2 * j + 1]))),
        "l"(b01));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(v1) : "l"(f32x2_pack(__uint_as_float(r[2 * j + 2]),
                                                              __uint_as_float(r[2 * j + 3]))),
        "l"(b23));
    const float2 f0 = f32x2_unpack(v0), f1 = f32x2_unpack(v1);
    asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(w[j]) : "f"(f0.y), "f"(f0.x));
    asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(w[j + 1]) : "f"(f1.y), "f"(f1.x));
  }
  if constexpr (W == 32) tc_st16(tmem + lanes + (uint32_t)(a_col + c0 / 2), w);
  else tc_st8(tmem + lanes + (uint32_t)(a_col + c0 / 2), w);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kFusedThreads, 1) actor_tc_fused_kernel(const TcLaunch p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const FusedLayout f = fused_layout(p.desc, p.tc_npad);
  unsigned char* feat = base + f.feat;
  float* sbias = reinterpret_cast<float*>(base + f.bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + f.bars);
  uint64_t* wbar = bars;          // weights resident
  uint64_t* ffull = bars + 1;     // [NB <= 4] feature tile ready (4 builder warps)
  uint64_t* ffree = bars + 5;     // [NB] feature tile consumed (MMA1 commit)
  // The block's chain runs in N halves (h = 0: D columns [0, n/2), 1: the
  // rest) so each epilogue's first half overlaps the MMAs of the second:
  uint64_t* d1h = bars + 9;       // [2] MMA1 N half h complete
  uint64_t* a2h = bars + 11;      // [2] epi1 chunk h done by every epilogue warp: A2 K
                                  //     columns of half h written, D1 half h drained
  uint64_t* d2h = bars + 13;      // [2] MMA2 N half h complete
  uint64_t* a3h = bars + 15;      // [2] epi2 chunk h done (A3 K half h, D2 half h drained)
  uint64_t* d3full = bars + 17;   // MMA3 complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n1 = p.tc_npad[0], n2 = p.tc_npad[1], n3 = p.tc_npad[2];
  const int nblocks = (p.ncols + kTcM - 1) / kTcM;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    mbar_init(wbar, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&ffull[i], 4);
      mbar_init(&ffree[i], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&d1h[h], 1);
      mbar_init(&d2h[h], 1);
      mbar_init(&a2h[h], kFusedEpi);
      mbar_init(&a3h[h], kFusedEpi);
    }
    mbar_init(d3full, 1);
    fence_mbar_init();
  }
  {  // biases (fp32) -> shared, zero past each layer's width
    const int nb[3] = {n1, n2, n3};
    int o = 0;
    for (int l = 0; l < 3; ++l) {
      const int out = p.desc.layer[l].out;
      const float* b = p.bias + p.desc.layer[l].b_off;
      for (int i = tid; i < nb[l]; i += blockDim.x) sbias[o + i] = i < out ? b[i] : 0.f;
      o += nb[l];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
#ifdef CYR_FUSED_PROF
  __shared__ long long trace[64];  // one steady-state block's event clocks (CTA 0)
  constexpr int kTraceBlock = 100;
#define CYR_TRACE(slot, it) \
  if ((it) == kTraceBlock && lane == 0) trace[slot] = clock64();
#endif
  const float* bias1 = sbias;
  const float* bias2 = sbias + n1;
  const float* bias3 = sbias + n1 + n2;

  constexpr int NB = kFusedGroups < 2 ? 2 : kFusedGroups;  // A1 tiles in flight
  if (warp == kFusedMmaWarp) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t total = f.w_bytes[0] + f.w_bytes[1] + f.w_bytes[2];
      mbar_expect_tx(wbar, total);
      for (int l = 0; l < 3; ++l)
        for (uint32_t c = 0; c < f.w_bytes[l]; c += 16384u) {
          const uint32_t nbytes = min(16384u, f.w_bytes[l] - c);
          bulk_g2s(base + f.w_off[l] + c, p.tc_blob + p.tc_off[l] + c, nbytes, wbar);
        }
    }
    __syncwarp();
    {  // the whole warp runs the issue loop; the tc_mma_* asm elect the issuing lane
      // The only CTA on the SM allocates all 512 columns, so the allocation
      // starts at lane 0, column 0.  With the base a compile-time 0 the MMA
      // operands are immediates and uniform-datapath adds; from the base read
      // out of shared memory ptxas re-broadcast every operand of every MMA
      // (R2UR.BROADCAST), ~100 cycles per N = 32 MMA instead of ~17.
      if (tmem != 0u) __trap();
      constexpr uint32_t tm = 0u;
      mbar_wait(wbar, 0);
      tc_fence_after();
      auto idesc = [](int n) {
        return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
               ((uint32_t)(kTcM >> 4) << 24);
      };
      const uint32_t id1 = idesc(n1 / 2), id2 = idesc(n2 / 2), id3 = idesc(n3);
      const uint32_t w1 = smem_u32(base + f.w_off[0]), w2 = smem_u32(base + f.w_off[1]),
                     w3 = smem_u32(base + f.w_off[2]);
      const uint32_t t2 = (uint32_t)n2 * 128u, t3 = (uint32_t)n3 * 128u;  // bytes per K tile
      // rows [n/2, n) of a SW128 weight image start (n/2/8) 1-KB row groups in
      const uint32_t w1b = w1 + (uint32_t)(n1 / 16) * 1024u, w2b = (uint32_t)(n2 / 16) * 1024u;
      const int k2 = n1 / 16, k3 = n2 / 16;  // K steps of MMA2 / MMA3
      int i = 0;
#ifdef CYR_FUSED_PROF
      const long long pstart = clock64();
#endif
      for (int b = blockIdx.x; b < nblocks; b += gridDim.x, ++i) {
        const int fb = i % NB;
        const uint32_t ph = (uint32_t)(i & 1);
        mbar_wait(&ffull[fb], (uint32_t)((i / NB) & 1));
        tc_fence_after();
#ifdef CYR_FUSED_PROF
        CYR_TRACE(0, i)
        CYR_TRACE(12, i - 1)
#endif
        // MMA1 (K = 64, one tile) in N halves
        const uint32_t a1 = smem_u32(feat + fb * kTcM * 128);
        tc_mma_ss_x4(tm, umma_desc_sw128(a1), umma_desc_sw128(w1), id1, 0);
        tc_commit_w(&d1h[0]);
        tc_mma_ss_x4(tm + (uint32_t)(n1 / 2), umma_desc_sw128(a1), umma_desc_sw128(w1b), id1, 0);
        tc_commit_w(&ffree[fb]);
        tc_commit_w(&d1h[1]);
        // MMA2 half 0 over K half 0 (A2 from epi1 chunk 0; it drained D1 half
        // 0, which D2 half 0 overwrites), then over K half 1 once epi1 chunk 1
        // is in, then half 1 over all of K: epi2 chunk 0 overlaps the last.
        CYR_FUSED_WAIT(&a2h[0], ph);
        tc_fence_after();
        for (int ks = 0; ks < k2 / 2; ks += 4)
          tc_mma_ts_x4(tm, tm + (uint32_t)(kFusedA2Col + ks * 8),
                       umma_desc_sw128(w2 + (uint32_t)(ks >> 2) * t2), id2, ks > 0 ? 1 : 0);
        CYR_FUSED_WAIT(&a2h[1], ph);
        tc_fence_after();
#ifdef CYR_FUSED_PROF
        CYR_TRACE(1, i)
#endif
        for (int ks = k2 / 2; ks < k2; ks += 4)
          tc_mma_ts_x4(tm, tm + (uint32_t)(kFusedA2Col + ks * 8),
                       umma_desc_sw128(w2 + (uint32_t)(ks >> 2) * t2), id2, 1);
        tc_commit_w(&d2h[0]);
        for (int ks = 0; ks < k2; ks += 4)
          tc_mma_ts_x4(tm + (uint32_t)(n2 / 2), tm + (uint32_t)(kFusedA2Col + ks * 8),
                       umma_desc_sw128(w2 + w2b + (uint32_t)(ks >> 2) * t2), id2, ks > 0 ? 1 : 0);
        tc_commit_w(&d2h[1]);
#ifdef CYR_FUSED_PROF
        CYR_TRACE(2, i)
#endif
        // MMA3 (the head) over K half 0 as soon as epi2 chunk 0 is in, then half 1
        CYR_FUSED_WAIT(&a3h[0], ph);
        tc_fence_after();
#ifdef CYR_FUSED_PROF
        CYR_TRACE(22, i)
#endif
        for (int ks = 0; ks < k3 / 2; ks += 4)
          tc_mma_ts_x4(tm + kFusedD3Col, tm + (uint32_t)(kFusedA3Col + ks * 8),
                       umma_desc_sw128(w3 + (uint32_t)(ks >> 2) * t3), id3, ks > 0 ? 1 : 0);
        CYR_FUSED_WAIT(&a3h[1], ph);
        tc_fence_after();
        for (int ks = k3 / 2; ks < k3; ks += 4)
          tc_mma_ts_x4(tm + kFusedD3Col, tm + (uint32_t)(kFusedA3Col + ks * 8),
                       umma_desc_sw128(w3 + (uint32_t)(ks >> 2) * t3), id3, 1);
#ifdef CYR_FUSED_PROF
        CYR_TRACE(23, i)
#endif
        tc_commit_w(d3full);
#ifdef CYR_FUSED_PROF
        CYR_TRACE(3, i)
#endif
      }
#ifdef CYR_FUSED_PROF
      if ((blockIdx.x == 0 || blockIdx.x == 77) && lane == 0)
        printf("MMA cta %d blocks %d: %lld cycles per block\n", blockIdx.x, i,
               (clock64() - pstart) / max(i, 1));
#endif
    }
    __syncwarp();
  } else if (warp >= kFusedEpi) {
    // ---------------------------------------------------- feature builders
    const int grp = (warp - kFusedEpi) >> 2, row = (tid - 32 * kFusedEpi) & 127;
    int i = 0;
    for (int b = blockIdx.x; b < nblocks; b += gridDim.x, ++i) {
      const int fb = i % NB;
      if (kFusedGroups > 1 && fb != grp) continue;
      if (i >= NB) mbar_wait(&ffree[fb], (uint32_t)(((i / NB) - 1) & 1));
#ifdef CYR_FUSED_PROF
      if (warp == kFusedEpi) { CYR_TRACE(60, i - 1) }
#endif
      tc_feature_tile(p, b * kTcM + row, 0, feat + fb * kTcM * 128, row);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ffull[fb]);
#ifdef CYR_FUSED_PROF
      if (warp == kFusedEpi) { CYR_TRACE(61, i - 1) }
#endif
    }
  } else {
    // ------------------------------------------------------------ epilogues
    // Every warp does its column chunk of N half 0, arrives, then half 1:
    // half 0 of each layer is complete (and its MMAs can start) while half 1
    // is still being converted.  Warp = (lane quarter, part): chunk columns
    // [h * n/2 + part * n/8, + n/8) of its 32 TMEM lanes.
    const int quarter = warp & 3, part = warp >> 2;
    const int cw1 = n1 / (2 * kFusedParts), cw2 = n2 / (2 * kFusedParts);  // 32 or 16
    auto chunk = [&](int cw, int c0, int a_col, const float* bias) {
      if (cw == 32) fused_epi_chunk<32>(tmem, quarter, c0, a_col, bias);
      else fused_epi_chunk<16>(tmem, quarter, c0, a_col, bias);
      tc_fence_before();
      __syncwarp();
    };
    const int out3 = p.desc.layer[2].out;
    const int row = quarter * 32 + lane;  // TMEM lane = column within the block
    const bool leader = warp == 0 && lane == 0;
    // Head output.  Right after MMA3 each warp reads 8 of D3's columns for
    // its 32 TMEM lanes (part p: logits [8p, 8p + 8)) into registers, then a
    // barrier: the next block's epi1 may overwrite those columns with A2.  The
    // logits are staged row-major in shared memory (the block's 128 x out3
    // fp32 = its contiguous slice of `raw`) and written by one bulk copy
    // while the next block's MMA2 runs.
    const int hc0 = part * 8;
    float hbias[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) hbias[j] = hc0 + j < n3 ? bias3[hc0 + j] : 0.f;
    float hv[8];
    auto head_read = [&]() {
      uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (hc0 < n3) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
              "=r"(r[6]), "=r"(r[7])
            : "r"(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(kFusedD3Col + hc0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) hv[j] = __uint_as_float(r[j]) + hbias[j];
      tc_fence_before();
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kFusedEpi) : "memory");  // every D3 read done
    };
    auto head_write = [&](int hb, int hi) {
      if (f.stage_bytes) {
        if (leader && hi > 0) bulk_wait_read<0>();  // the previous block's store has read the stage
        asm volatile("bar.sync 2, %0;" ::"n"(32 * kFusedEpi) : "memory");
        const uint32_t st = smem_u32(base + f.stage) + (uint32_t)(row * out3 + hc0) * 4u;
        if ((out3 & 3) == 0 && hc0 + 8 <= out3) {
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(st), "f"(hv[0]),
                       "f"(hv[1]), "f"(hv[2]), "f"(hv[3]));
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(st + 16u), "f"(hv[4]),
                       "f"(hv[5]), "f"(hv[6]), "f"(hv[7]));
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (hc0 + j < out3) asm volatile("st.shared.f32 [%0], %1;" ::"r"(st + 4u * j), "f"(hv[j]));
        }
        fence_proxy_async_smem();
        asm volatile("bar.sync 2, %0;" ::"n"(32 * kFusedEpi) : "memory");
        const int valid = min(kTcM, p.ncols - hb * kTcM);
        const uint32_t bytes = (uint32_t)valid * (uint32_t)out3 * 4u;
        float* dst = p.raw + (long long)hb * kTcM * out3;
        if (bytes % 16u == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
          if (leader) {
            bulk_s2g(dst, base + f.stage, bytes);
            bulk_commit();
          }
        } else {  // ragged last block / unaligned output: coalesced word copy
          const float* s0 = reinterpret_cast<const float*>(base + f.stage);
          for (int e = tid; e < valid * out3; e += 32 * kFusedEpi) dst[e] = s0[e];
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kFusedEpi) : "memory");
        }
      } else {  // no room for the stage: direct stores
        const int col = hb * kTcM + row;
        if (col < p.ncols)
          for (int j = 0; j < 8; ++j)
            if (hc0 + j < out3) p.raw[(long long)col * out3 + hc0 + j] = hv[j];
      }
    };
    int i = 0, prev = -1;
    for (int b = blockIdx.x; b < nblocks; b += gridDim.x, ++i) {
      const uint32_t ph = (uint32_t)(i & 1);
      for (int h = 0; h < 2; ++h) {  // epi1: D1 -> A2
        CYR_FUSED_WAIT(&d1h[h], ph);
        tc_fence_after();
#ifdef CYR_FUSED_PROF
        if (warp == 0) { CYR_TRACE(4 + h, i) }
#endif
        chunk(cw1, h * (n1 / 2) + part * cw1, kFusedA2Col, bias1);
        if (lane == 0) mbar_arrive(&a2h[h]);
#ifdef CYR_FUSED_PROF
        if (warp == 0) { CYR_TRACE(6 + h, i) }
#endif
      }
      if (prev >= 0) head_write(prev, i - 1);  // the previous block's logits, during MMA2
      for (int h = 0; h < 2; ++h) {  // epi2: D2 -> A3
        CYR_FUSED_WAIT(&d2h[h], ph);
        tc_fence_after();
#ifdef CYR_FUSED_PROF
        if (warp == 0) { CYR_TRACE(8 + h, i) }
#endif
        chunk(cw2, h * (n2 / 2) + part * cw2, kFusedA3Col, bias2);
        if (lane == 0) mbar_arrive(&a3h[h]);
#ifdef CYR_FUSED_PROF
        if (warp == 0) { CYR_TRACE(10 + h, i) }
#endif
      }
      CYR_FUSED_WAIT(d3full, ph);
      tc_fence_after();
#ifdef CYR_FUSED_PROF
      if (warp == 0) { CYR_TRACE(20, i) }
#endif
      head_read();
#ifdef CYR_FUSED_PROF
      if (warp == 0) { CYR_TRACE(21, i) }
#endif
      prev = b;
    }
    if (prev >= 0) head_write(prev, i - 1);
    if (leader && f.stage_bytes) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
#ifdef CYR_FUSED_PROF
  if (tid == 0 && blockIdx.x == 0 && nblocks > kTraceBlock * (int)gridDim.x &&
      atomicAdd(&g_fused_trace_launch, 1) == 1) {  // one launch (the 2nd large one) prints
    const long long t0 = trace[0];
    printf("TRACE cta 0 block %d (clocks after its features are in): MMA2 K-half 1 start %lld, "
           "MMA2 issued %lld, MMA3 K-half 0 start %lld, MMA3 issued %lld, next block %lld | "
           "epi1 d1h %lld/%lld done %lld/%lld | epi2 d2h %lld/%lld done %lld/%lld | head d3 seen "
           "%lld done %lld\n", kTraceBlock, trace[1] - t0, trace[2] - t0, trace[22] - t0,
           trace[23] - t0, trace[12] - t0, trace[4] - t0, trace[5] - t0, trace[6] - t0,
           trace[7] - t0, trace[8] - t0, trace[9] - t0, trace[10] - t0, trace[11] - t0,
           trace[20] - t0, trace[21] - t0);
    printf("TRACE cta 0 builder: next block's features %lld .. %lld\n", trace[60] - t0,
           trace[61] - t0);
  }
#endif
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------- wide layers
// Actors wider than one MMA tile (cfg5: 3 x 1024) run layer by layer, each
// layer a persistent warp-specialised tcgen05 GEMM:
//   warp 8  producer: TMA bulk copies of {A tile 16 KB, B tile <= 32 KB}
//           K-tile stages into a ring (FIRST: streams only B);
//   warps 10-13 (FIRST only) feature builders: thread = row of the block's
//           feature A tile, double-buffered across column blocks;
//   warp 9  MMA issuer (one lane): D[128 x 256] per (column block, n tile)
//           into one of two TMEM accumulators (2 x 256 columns);
//   warps 0-3 (FIRST: 0-7) epilogue, one (two) groups of 4 warps (warp w
//           reads TMEM lane quarter w % 4), group g taking its share of the
//           accumulator columns: tcgen05.ld, bias (+ReLU), bf16, into the
//           group's two 16 KB staging images, TMA bulk store (LAST: fp32
//           logits raw[col][2E]).  The K = 64 first layer gets two groups:
//           it is epilogue-bound (4 MMAs per n tile against 4 images of
//           stores), as does any layer with <= 4 K tiles (cfg2's 256 x 256);
//           deeper K keeps the shared memory for the ring.
// Each CTA walks column blocks with a grid stride and every n tile of a block
// back to back, so the block's A tiles are L2-hot for tiles 2..4 and the
// epilogue of one tile overlaps the MMAs of the next.  With fewer blocks
// than SMs (the top tree levels) the n tiles of a block are split over
// `split` CTAs instead, so a small level is not one SM streaming all weights.  Activations
// live in HBM as the SW128 K-major images the MMA reads: [col block][k tile]
// [128 x 64] bf16, written by the previous layer's epilogue.
constexpr int kWideThreads = 320;       // + 128 feature builders for the first layer
constexpr int kWideFirstThreads = 448;
constexpr int kWideImage = kTcM * 128;  // one [128 x 64] bf16 image, 16 KB
constexpr int kWideMaxSlots = 8;

struct TcWideLaunch {
  TcLaunch base;  // features / raw / Mode-T fields
  int l, in, out, npad;
  int kt;          // K tiles of this layer (1 for the first)
  int nts;         // n tiles of 256
  int ncb;         // column blocks of 128
  int nslots;      // ring depth
  int split;       // CTAs per column block (n tiles divided between them)
  uint32_t slot_bytes, a_bytes;  // per stage (a_bytes = 0 for the first layer)
  long long w_off;  // this layer's images: [n tile][k tile][256 x 128 B]
  long long b_stride;  // bytes per k tile: 256 x 128, or npad x 128 for a single n tile
  const unsigned char* act_in;  // [ncb][kt][16 KB]
  unsigned char* act_out;       // [ncb][ceil(out/64)][16 KB]
};

__device__ __forceinline__ void epi_sync(int grp) {  // the 128 threads of one epilogue group
  asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
}

template <bool FIRST, bool LAST, int EG>
__global__ void __launch_bounds__(kWideFirstThreads, 1) actor_tc_wide_kernel(const TcWideLaunch q) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* ring = base;
  unsigned char* feat = ring + (size_t)q.nslots * q.slot_bytes;  // FIRST: 2 x 16 KB
  // EG epilogue groups of 4 warps: 2 where the layer is epilogue-bound
  // (few K tiles per n tile), 1 where the MMAs dominate (ring depth first)
  unsigned char* stg = feat + (FIRST ? 2 * kWideImage : 0);      // !LAST: EG x 2 x 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + (LAST ? 0 : EG * 2 * kWideImage));
  uint64_t* full = bars;
  uint64_t* freeb = full + kWideMaxSlots;
  uint64_t* tfull = freeb + kWideMaxSlots;
  uint64_t* tempty = tfull + 2;
  uint64_t* ffull = tempty + 2;
  uint64_t* ffree = ffull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ffree + 2);
  const TcLaunch& p = q.base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = q.nslots;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&freeb[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4 * EG);
      mbar_init(&ffull[i], 4);
      mbar_init(&ffree[i], 1);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int last_nt_rows = q.npad - (q.nts - 1) * 256;
  // this CTA: column blocks cb0, cb0 + cbs, ...; n tiles [nt0, nt1) of each
  const int sp = blockIdx.x % q.split;
  const int cb0 = blockIdx.x / q.split, cbs = gridDim.x / q.split;
  const int nt0 = sp * q.nts / q.split, nt1 = (sp + 1) * q.nts / q.split;

  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      long long st = 0;
      for (int cb = cb0; cb < q.ncb; cb += cbs) {
        for (int nt = nt0; nt < nt1; ++nt) {
          const uint32_t b_bytes = (uint32_t)(nt == q.nts - 1 ? last_nt_rows : 256) * 128;
          for (int t = 0; t < q.kt; ++t, ++st) {
            const int slot = (int)(st % NS);
            if (st >= NS) mbar_wait(&freeb[slot], (uint32_t)(((st / NS) - 1) & 1));
            unsigned char* dst = ring + (size_t)slot * q.slot_bytes;
            mbar_expect_tx(&full[slot], q.a_bytes + b_bytes);
            if (!FIRST)
              bulk_g2s(dst, q.act_in + ((long long)cb * q.kt + t) * kWideImage, kWideImage,
                       &full[slot]);
            bulk_g2s(dst + q.a_bytes,
                     p.tc_blob + q.w_off + ((long long)nt * q.kt + t) * q.b_stride, b_bytes,
                     &full[slot]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 10) {
    // ---------------------------------------- feature builders (first layer)
    if (FIRST) {
      const int row = tid - 320;
      int i = 0;
      for (int cb = cb0; cb < q.ncb; cb += cbs, ++i) {
        const int fb = i & 1;
        if (i >= 2) mbar_wait(&ffree[fb], (uint32_t)(((i >> 1) - 1) & 1));
        tc_feature_tile(p, cb * kTcM + row, 0, feat + fb * kWideImage, row);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ffull[fb]);
      }
    }
  } else if (warp == 9) {
    // ---------------------------------------------------------- MMA issuer
    {  // whole warp: one asm per K tile elects the issuing lane (tc_mma_ss_x4)
      long long st = 0;
      int a = 0, i = 0;
      for (int cb = cb0; cb < q.ncb; cb += cbs, ++i) {
        const int fb = i & 1;
        if (FIRST) {
          mbar_wait(&ffull[fb], (uint32_t)((i >> 1) & 1));
          tc_fence_after();
        }
        for (int nt = nt0; nt < nt1; ++nt, ++a) {
          const int acc = a & 1, u = a >> 1;
          if (u >= 1) {
            mbar_wait(&tempty[acc], (uint32_t)((u - 1) & 1));
            tc_fence_after();
          }
          const int rows_n = nt == q.nts - 1 ? last_nt_rows : 256;
          const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                 ((uint32_t)(rows_n >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
          const uint32_t d = tmem + (uint32_t)(acc * 256);
          for (int t = 0; t < q.kt; ++t, ++st) {
            const int slot = (int)(st % NS);
            mbar_wait(&full[slot], (uint32_t)((st / NS) & 1));
            tc_fence_after();
            const uint32_t s_addr = smem_u32(ring + (size_t)slot * q.slot_bytes);
            const uint32_t a_addr = FIRST ? smem_u32(feat + fb * kWideImage) : s_addr;
            const uint32_t b_addr = s_addr + q.a_bytes;
            tc_mma_ss_x4(d, umma_desc_sw128(a_addr), umma_desc_sw128(b_addr), idesc, t > 0 ? 1 : 0);
            tc_commit_w(&freeb[slot]);
          }
          tc_commit_w(&tfull[acc]);
        }
        if (FIRST) tc_commit_w(&ffree[fb]);
      }
    }
    __syncwarp();
  } else if (warp < 4 * EG) {
    // ------------------------------------------------------------ epilogue
    const float* bias = p.bias + p.desc.layer[q.l].b_off;
    const int kt_next = (q.out + 63) / 64;
    const int grp = warp >> 2, wq = warp & 3;  // group; TMEM lane quarter
    const int row = tid & 127;                 // = TMEM lane = column within the block
    const bool leader = row == 0;
    int a = 0, img = 0;
    for (int cb = cb0; cb < q.ncb; cb += cbs) {
      const int col = cb * kTcM + row;
      for (int nt = nt0; nt < nt1; ++nt, ++a) {
        const int acc = a & 1, u = a >> 1;
        mbar_wait(&tfull[acc], (uint32_t)(u & 1));
        tc_fence_after();
        const int rows_n = nt == q.nts - 1 ? last_nt_rows : 256;
        for (int n0 = grp * (256 / EG); n0 < min(rows_n, (grp + 1) * (256 / EG)); n0 += 64) {
          uint32_t r[64];
          const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(acc * 256 + n0);
          tc_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tc_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          const int o0 = nt * 256 + n0;
          if (LAST) {
            if (col < p.ncols) {
              float* dst = p.raw + (long long)col * q.out;
              for (int j = 0; j < 64; ++j)
                if (o0 + j < q.out) dst[o0 + j] = __uint_as_float(r[j]) + bias[o0 + j];
            }
          } else {
            const int sb = img & 1;
            if (leader) bulk_wait_read<1>();  // the store that last used this image has read it
            epi_sync(grp);
            unsigned char* sp = stg + (grp * 2 + sb) * kWideImage;
            const uint32_t spa = smem_u32(sp);
            // whole 8-output groups inside the layer with a 16-byte aligned
            // bias: two float4 loads (uniform broadcast) per group instead of
            // eight scalar ones, packed add + ReLU-folded convert (the fused
            // MLP's epilogue), explicit st.shared
            const bool vec = o0 + 64 <= q.out && ((reinterpret_cast<uintptr_t>(bias + o0) & 15u) == 0);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              uint32_t w[4];
              if (vec) {
                const float4 ba = __ldg(reinterpret_cast<const float4*>(bias + o0 + c * 8));
                const float4 bb = __ldg(reinterpret_cast<const float4*>(bias + o0 + c * 8 + 4));
                const float bv[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  unsigned long long v;
                  asm("add.rn.f32x2 %0, %1, %2;"
                      : "=l"(v)
                      : "l"(f32x2_pack(__uint_as_float(r[c * 8 + 2 * h]),
                                       __uint_as_float(r[c * 8 + 2 * h + 1]))),
                        "l"(f32x2_pack(bv[2 * h], bv[2 * h + 1])));
                  const float2 f = f32x2_unpack(v);
                  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(w[h]) : "f"(f.y), "f"(f.x));
                }
              } else {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  const int j = c * 8 + 2 * h, o = o0 + j;
                  float v0 = o < q.out ? __uint_as_float(r[j]) + bias[o] : 0.f;
                  float v1 = o + 1 < q.out ? __uint_as_float(r[j + 1]) + bias[o + 1] : 0.f;
                  v0 = v0 > 0.f ? v0 : 0.f;
                  v1 = v1 > 0.f ? v1 : 0.f;
                  const __nv_bfloat162 pr = __floats2bfloat162_rn(v0, v1);
                  w[h] = *reinterpret_cast<const uint32_t*>(&pr);
                }
              }
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(spa + sw128_offset(row, c * 8)),
                           "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]));
            }
            fence_proxy_async_smem();
            epi_sync(grp);
            if (leader) {
              bulk_s2g(q.act_out + ((long long)cb * kt_next + (o0 >> 6)) * kWideImage, sp,
                       kWideImage);
              bulk_commit();
            }
            ++img;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
    }
    if (!LAST && leader) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace cyr

size_t cyr_tc_smem_bytes() {
  return 1024 + (size_t)cyr::kTcMaxKt * cyr::kTcM * 128 + (size_t)cyr::kTcSlots * cyr::kTcSlotBytes +
         (2 * cyr::kTcSlots + 1) * 8 + 16;
}

int cyr_launch_actor_tc(const cyr::ActorDesc& desc, const unsigned char* tc_blob,
                        const long long* tc_off, const int* tc_npad, const float* bias_blob,
                        const int32_t* alloc, int S, int E, int N, int cap, float* raw,
                        int mode_t, const int32_t* mcs, const int16_t* node, int M, int tau,
                        int parents, long long nodes_per_slot, long long parent_off, int epad,
                        double mcs_scale, cudaStream_t stream, int parent_base) {
  cyr::TcLaunch p{};
  p.desc = desc;
  for (int l = 0; l < desc.n_layers; ++l) {
    if (desc.layer[l].in > 64 * cyr::kTcMaxKt || tc_npad[l] > 256) return CYR_UNSUPPORTED;
    p.tc_off[l] = tc_off[l];
    p.tc_npad[l] = tc_npad[l];
  }
  p.tc_blob = tc_blob;
  p.bias = bias_blob;
  p.alloc = alloc;
  p.raw = raw;
  p.S = S;
  p.E = E;
  p.N = N;
  p.cap = cap;
  const long long ncols = mode_t ? (long long)S * parents * cap : (long long)S * cap;
  if (ncols <= 0) return CYR_OK;
  if (ncols >= (1ll << 31)) return CYR_UNSUPPORTED;
  p.ncols = (int)ncols;
  p.mode_t = mode_t;
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
  const size_t smem = cyr_tc_smem_bytes();
  static cyr::AttrCache configured;
  if (!cyr::ensure_func_attr(configured, (int)smem, [&] {
        return cudaFuncSetAttribute(cyr::actor_tc_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess;
      }))
    return CYR_CUDA_ERROR;
  const int blocks = (p.ncols + cyr::kTcM - 1) / cyr::kTcM;
  cyr::actor_tc_kernel<<<blocks, cyr::kTcThreads, smem, stream>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

int cyr_launch_actor_tc_layer(const cyr::ActorDesc& desc, const unsigned char* tc_blob,
                              long long w_off, int npad, int l, const float* bias_blob,
                              const int32_t* alloc, int S, int E, int N, int cap, float* raw,
                              const unsigned char* act_in, unsigned char* act_out, int mode_t,
                              const int32_t* mcs, const int16_t* node, int M, int tau,
                              int parents, long long nodes_per_slot, long long parent_off,
                              int epad, double mcs_scale, cudaStream_t stream,
                              int parent_base) {
  cyr::TcWideLaunch q{};
  cyr::TcLaunch& p = q.base;
  p.desc = desc;
  p.tc_blob = tc_blob;
  p.bias = bias_blob;
  p.alloc = alloc;
  p.raw = raw;
  p.S = S;
  p.E = E;
  p.N = N;
  p.cap = cap;
  const long long ncols = mode_t ? (long long)S * parents * cap : (long long)S * cap;
  if (ncols <= 0) return CYR_OK;
  if (ncols >= (1ll << 31)) return CYR_UNSUPPORTED;
  p.ncols = (int)ncols;
  p.mode_t = mode_t;
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
  const cyr::LayerDesc& L = desc.layer[l];
  const bool first = l == 0, last = l == desc.n_layers - 1;
  if (first && last) return CYR_UNSUPPORTED;
  if (first && L.in > 64) return CYR_UNSUPPORTED;
  q.l = l;
  q.in = L.in;
  q.out = L.out;
  q.npad = npad;
  q.kt = first ? 1 : (L.in + 63) / 64;
  q.nts = (npad + 255) / 256;
  q.ncb = (int)((ncols + cyr::kTcM - 1) / cyr::kTcM);
  q.w_off = w_off;
  q.b_stride = (q.nts > 1 ? 256 : npad) * 128ll;
  q.act_in = act_in;
  q.act_out = act_out;
  q.a_bytes = first ? 0u : (uint32_t)cyr::kWideImage;
  const int b_rows = std::min(256, npad);
  q.slot_bytes = (uint32_t)((q.a_bytes + b_rows * 128 + 1023) / 1024 * 1024);
  const int eg = (first || q.kt <= 4) ? 2 : 1;  // epilogue groups (see the kernel)
  const size_t fixed = 1024 + (first ? 2 * cyr::kWideImage : 0) +
                       (last ? 0 : eg * 2 * cyr::kWideImage) +
                       (4 * cyr::kWideMaxSlots + 16) * 8 + 16;
  int max_smem = 0, sms = 0;
  {
    const int dev = cyr::current_device_ordinal();
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  q.nslots = (int)std::min<size_t>(cyr::kWideMaxSlots, (max_smem - fixed) / q.slot_bytes);
  if (q.nslots < 2) return CYR_UNSUPPORTED;
  const size_t smem = fixed + (size_t)q.nslots * q.slot_bytes;
  q.split = std::max(1, std::min(q.nts, sms / std::max(q.ncb, 1)));
  const dim3 grid((unsigned)(std::min(q.ncb, sms / q.split) * q.split));
#define CYR_WIDE(F, LST, G)                                                                    \
  do {                                                                                         \
    if (cudaFuncSetAttribute(cyr::actor_tc_wide_kernel<F, LST, G>,                             \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem) !=         \
        cudaSuccess)                                                                           \
      return CYR_CUDA_ERROR;                                                                   \
    cyr::actor_tc_wide_kernel<F, LST, G>                                                       \
        <<<grid, F ? cyr::kWideFirstThreads : cyr::kWideThreads, smem, stream>>>(q);           \
  } while (0)
  if (first) CYR_WIDE(true, false, 2);
  else if (last) CYR_WIDE(false, true, 1);
  else if (eg == 2) CYR_WIDE(false, false, 2);
  else CYR_WIDE(false, false, 1);
#undef CYR_WIDE
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}

// the fused narrow kernel applies: 3 layers, first K <= 64, hidden widths
// padded to multiples of 64 (<= 256), head <= 64 outputs, fits shared memory
bool cyr_tc_fused_applies(const cyr::ActorDesc& desc, const int* tc_npad) {
  if (desc.n_layers != 3 || desc.layer[0].in > 64) return false;
  for (int l = 0; l < 2; ++l)  // hidden widths: whole 32-column epilogue chunks per part
    if (tc_npad[l] > 256 || tc_npad[l] % (32 * cyr::kFusedParts) != 0) return false;
  if (tc_npad[2] > 64) return false;
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                         cyr::current_device_ordinal());
  return cyr::fused_layout(desc, tc_npad).total <= (uint32_t)max_smem;
}

int cyr_launch_actor_tc_fused(const cyr::ActorDesc& desc, const unsigned char* tc_blob,
                              const long long* tc_off, const int* tc_npad, const float* bias_blob,
                              const int32_t* alloc, int S, int E, int N, int cap, float* raw,
                              int mode_t, const int32_t* mcs, const int16_t* node, int M, int tau,
                              int parents, long long nodes_per_slot, long long parent_off,
                              int epad, double mcs_scale, int sm_count, cudaStream_t stream,
                              int parent_base) {
  if (!cyr_tc_fused_applies(desc, tc_npad)) return CYR_UNSUPPORTED;
  cyr::TcLaunch p{};
  p.desc = desc;
  for (int l = 0; l < desc.n_layers; ++l) {
    p.tc_off[l] = tc_off[l];
    p.tc_npad[l] = tc_npad[l];
  }
  p.tc_blob = tc_blob;
  p.bias = bias_blob;
  p.alloc = alloc;
  p.raw = raw;
  p.S = S;
  p.E = E;
  p.N = N;
  p.cap = cap;
  const long long ncols = mode_t ? (long long)S * parents * cap : (long long)S * cap;
  if (ncols <= 0) return CYR_OK;
  if (ncols >= (1ll << 31)) return CYR_UNSUPPORTED;
  p.ncols = (int)ncols;
  p.mode_t = mode_t;
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
  const size_t smem = cyr::fused_layout(desc, tc_npad).total;
  static cyr::AttrCache configured;
  if (!cyr::ensure_func_attr(configured, (int)smem, [&] {
        return cudaFuncSetAttribute(cyr::actor_tc_fused_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess;
      }))
    return CYR_CUDA_ERROR;
  const int nblocks = (p.ncols + cyr::kTcM - 1) / cyr::kTcM;
  const int grid = std::min(nblocks, std::max(1, sm_count));
  cyr::actor_tc_fused_kernel<<<grid, cyr::kFusedThreads, smem, stream>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}
