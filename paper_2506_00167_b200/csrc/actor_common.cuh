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
