// actor_common.cuh — the K2 launch record and the actor's input features,
// shared by the fused batch kernels (actor.cu) and the layer-GEMM path
// (actor_gemm.cu).
#pragma once

#include "projection.cuh"

namespace cyr {

struct ActorLaunch {
  ActorDesc desc;
  const void* blob;
  const int32_t* alloc;
  void* raw;
  int S, E, N, cap, ncols;
  int stages;
  // fused single-slot path (K2 -> K3 in one cluster launch)
  const double* eps;
  int L;
  int32_t* cb;       // device codebook [S][cap+1][E]
  int32_t* cb_host;  // optional mapped-host copy of the codebook
  int32_t* status;
  unsigned long long* trace;  // CYR_TRACE phase stamps (rank 0), or null
  int inline_inputs;          // alloc / eps come from the SlotInline parameter
  // Mode T (actor on arrival-tree node states), batch kernel only
  int mode_t;
  const int16_t* node;        // node states [S][nodes][epad]
  const int32_t* mcs;         // [S][E]
  long long nodes_per_slot;
  long long parent_off;       // node offset of the first parent of this launch, -1 for the root
  int parents, tau, M, epad;
  int parent_base;            // level index of the first parent (subtree shards; digits -> arrivals)
  double mcs_scale;
  // column inputs (tiled kernel only): kcol -> column c is [alloc[c]/N, kcol[c]/cap]
  // (sac.critic_targets, sac.py:190-192); x -> explicit float64 features [c][in]
  const int32_t* kcol;
  const double* x;
};

// Mode-T actor input for column (slot s, parent q, branch k) — feature i of
// [n/N (E), k/cap, cum/N (E), mcs/mcs_scale (E), arrivals/(M*cap), (tau-1)/M].
// With zero weights on the last 2E+2 inputs this is exactly the Mode-R
// column [n/N, k/cap] (sac.py:344-346): the zero-pad bridge.
__device__ __forceinline__ double mode_t_feature(const ActorLaunch& p, int col, int i) {
  const int k = col % p.cap + 1;
  const int g = col / p.cap;
  const int s = g / p.parents;
  const int q = g - s * p.parents;
  const int E = p.E;
  if (i < E) return (double)p.alloc[(long long)s * E + i] / (double)p.N;
  if (i == E) return (double)k / (double)p.cap;
  if (i <= 2 * E) {
    if (p.parent_off < 0) return 0.0;
    const long long rec = (long long)s * p.nodes_per_slot + p.parent_off + q;
    return (double)p.node[rec * p.epad + (i - E - 1)] / (double)p.N;
  }
  if (i <= 3 * E) return (double)p.mcs[(long long)s * E + (i - 2 * E - 1)] / p.mcs_scale;
  if (i == 3 * E + 1) {
    int arrivals = 0, x = p.parent_base + q;
    for (int d = 1; d < p.tau; ++d) {
      arrivals += x % (p.cap + 1);
      x /= (p.cap + 1);
    }
    return (double)arrivals / (double)(p.M * p.cap);
  }
  return (double)(p.tau - 1) / (double)p.M;
}

// Packed fp32 pairs for FFMA2 (sm_100: fma.rn.f32x2, two IEEE fma.rn per
// instruction, so each lane's result is bit-identical to fmaf): the SIMT
// actor kernels are issue-bound, and one FFMA2 with a broadcast scalar
// operand (ptxas folds {a, a} into the instruction) issues two FMAs.
__device__ __forceinline__ unsigned long long f32x2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f32x2_unpack(unsigned long long v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return make_float2(lo, hi);
}
// acc.{lo,hi} = fma(a, b.{lo,hi}, acc.{lo,hi})
__device__ __forceinline__ void ffma2_bcast(unsigned long long& acc, float a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(f32x2_pack(a, a)), "l"(b));
}

// One input row of an 8-output x NC-column register tile:
// acc[a][b] = fma(w[a], x[b], acc[a][b]); fp32 column pairs go through FFMA2.
template <int NC>
__device__ __forceinline__ void fma_tile_row(float (&acc)[8][NC], const float (&w)[8],
                                             const float (&x)[NC]) {
  if constexpr (NC % 2 == 0) {
#pragma unroll
    for (int q = 0; q < NC / 2; ++q) {
      const unsigned long long xq = f32x2_pack(x[2 * q], x[2 * q + 1]);
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        unsigned long long c = f32x2_pack(acc[a][2 * q], acc[a][2 * q + 1]);
        ffma2_bcast(c, w[a], xq);
        const float2 v = f32x2_unpack(c);
        acc[a][2 * q] = v.x;
        acc[a][2 * q + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < NC; ++b) acc[a][b] = fmaf(w[a], x[b], acc[a][b]);
  }
}
template <int NC>
__device__ __forceinline__ void fma_tile_row(double (&acc)[8][NC], const double (&w)[8],
                                             const double (&x)[NC]) {
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < NC; ++b) acc[a][b] = fma(w[a], x[b], acc[a][b]);
}

// Input feature i of batch column col, float64 (rounded to the actor's
// precision by the caller):
//   explicit x [col][in]                                      (any MLP)
//   kcol: [alloc[col]/N, kcol[col]/cap]                       (sac.py:190-192)
//   Mode T: mode_t_feature                                    (node states)
//   Mode R: [alloc[s]/N, j/cap], s = col / cap, j = col % cap + 1 (sac.py:344-346)
__device__ __forceinline__ double column_feature(const ActorLaunch& p, int col, int i) {
  if (p.x) return p.x[(long long)col * p.desc.layer[0].in + i];
  if (p.mode_t) return mode_t_feature(p, col, i);
  const int s = p.kcol ? col : col / p.cap;
  const int j = p.kcol ? p.kcol[col] : col % p.cap + 1;
  return (i < p.E) ? (double)p.alloc[(long long)s * p.E + i] / (double)p.N
                   : (double)j / (double)p.cap;
}

}  // namespace cyr
