// actor_gemm.cu — K2 for WIDE fp32 actors (cfg5: 3 x 1024) on large column
// batches: the MLP layer by layer as SIMT SGEMMs over HBM activations.
//
// Why: the fused tiled kernel (actor.cu) keeps a CTA's activations for all
// layers in shared memory, so a 1024-wide actor leaves room for only 8
// columns per CTA and every CTA re-streams all 8 MiB of weights for them.
// Here each layer is one GEMM
//     Y[out][cols] = relu(Wt^T[out][K] . X[K][cols] + b)
// with X / Y fp32 in HBM ([feature][column], ldx = columns rounded to 128):
// a 128-output x 128-column CTA tile reuses every weight over 128 columns
// and every activation over 128 outputs.
//
// Numerics are the fused kernel's, bit for bit: the first layer's inputs
// are the same float64 features rounded to fp32 (column_feature), each
// output is ONE fp32 FMA chain over k = 0..K-1 in order from 0 (zero-padded
// k add exact zeros), then + bias, then ReLU; the last layer writes the
// logits as raw[col][out].
//
// Tile: 256 threads, 8 warps as 4 (outputs) x 2 (columns); a thread owns 8
// outputs x 8 columns (64 accumulators, packed in column pairs: 32 FFMA2 per
// k instead of 64 FFMA — the kernel is issue-bound), both split as {+0..3, +16/32..}
// so each of its four LDS.128 per k reads, across the warp, contiguous
// 16-byte chunks (one shared-memory wavefront each).  K advances in 16-row
// stages through a 3-deep cp.async ring (16 KB per stage), 2 CTAs per SM.
#include "actor_common.cuh"

#include <algorithm>
#include <type_traits>
#include <cstdlib>

namespace cyr {

constexpr int kGemmBM = 128, kGemmBN = 128, kGemmBK = 16, kGemmStages = 3;
constexpr int kGemmThreads = 256;
// narrow layers (the 2E-logit head, out <= 32): 32 outputs x 512 columns
constexpr int kHeadBM = 32, kHeadBN = 512;
template <int BM, int BN>
constexpr int stage_floats() { return kGemmBK * (BM + BN); }
// activation row stride: columns rounded to the widest tile, plus 32 floats
// so consecutive feature rows do not alias the same L2 partitions
inline int gemm_ldx(long long ncols) {
  return (int)((ncols + kHeadBN - 1) / kHeadBN * kHeadBN + 32);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = smem_u32(smem);
  const int bytes = valid ? 16 : 0;  // 0: zero-fill (out-of-range rows / outputs)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// X0[k][ldx] = (float)feature(col, k), zero for k >= in or col >= ncols
__global__ void __launch_bounds__(256) gemm_features_kernel(const ActorLaunch p, float* X, int ldx,
                                                            int kpad) {
  const long long n = (long long)kpad * ldx;
  const int in0 = p.desc.layer[0].in;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(idx / ldx), col = (int)(idx % ldx);
    X[idx] = (k < in0 && col < p.ncols) ? (float)column_feature(p, col, k) : 0.f;
  }
}

// The same X0, one thread per column group (the cap branch columns of one
// slot or Mode-T parent): every feature but k/cap is shared by the group, so
// it is evaluated once per group instead of once per column (the element
// kernel above spends its time on per-element index decoding); each thread
// writes its cap consecutive columns, a warp 32*cap contiguous floats per
// feature row.  Same float64 expressions (column_feature), same bits.
__global__ void __launch_bounds__(256) gemm_features_group_kernel(const ActorLaunch p, float* X,
                                                                  int ldx, int kpad) {
  const int cap = p.cap;
  const long long groups = (ldx + cap - 1) / cap;
  const int in0 = p.desc.layer[0].in;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
       g += (long long)gridDim.x * blockDim.x) {
    const long long c0 = g * cap;
    const bool live = c0 < p.ncols;
    for (int i = 0; i < kpad; ++i) {
      float* row = X + (long long)i * ldx + c0;
      const bool shared = i != p.E;
      const float v = (live && i < in0 && shared) ? (float)column_feature(p, (int)c0, i) : 0.f;
      for (int k = 0; k < cap; ++k) {
        const long long col = c0 + k;
        if (col >= ldx) break;
        float x = 0.f;
        if (col < p.ncols && i < in0) x = shared ? v : (float)column_feature(p, (int)col, i);
        row[k] = x;
      }
    }
  }
}

// One layer: K rows of X (K a multiple of 16 within ldx's allocation), Wt
// [K_w][ldw] (rows >= K_w read as zero), out outputs.  CTA tile BM outputs
// x BN columns, 8 warps as (BM/32) x (BN/64).
//
// OPT < 8 (the narrow head, BM = 32, out <= 4*OPT): a thread owns OPT
// consecutive outputs oy*OPT + {0..OPT-1} instead of 8 interleaved ones, so a
// 2E = 20-logit head runs 5 outputs per thread with no padded rows (the 8-row
// mapping spent 37.5 % of its FMAs on rows 20..31).  Same FMA chain per
// output, same bits.
template <int BM, int BN, bool LAST, int OPT = 8>
__global__ void __launch_bounds__(kGemmThreads, 2)
    sgemm_layer_kernel(const float* __restrict__ Wt, int ldw, int Kw, const float* __restrict__ bias,
                       const float* __restrict__ X, int ldx, int K, int out,
                       float* __restrict__ Y, int ldy, float* __restrict__ raw, int ncols) {
  static_assert((BM / 32) * (BN / 64) == kGemmThreads / 32, "8 warps");
  static_assert(OPT == 8 || (BM == 32 && LAST), "compact outputs: head only");
  constexpr int SF = stage_floats<BM, BN>();
  extern __shared__ __align__(16) float gsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int o0 = blockIdx.y * BM, c0 = blockIdx.x * BN;
  const int wy = warp / (BN / 64), wx = warp % (BN / 64);
  const int oy = lane >> 3, cx = lane & 7;
  // this thread's outputs: ob + {0..3} and ob + 16 + {0..3}; columns: cb + {0..3}, cb + 32 + {0..3}
  const int ob = wy * 32 + oy * 4, cb = wx * 64 + cx * 4;

  auto load_stage = [&](int kt, int buf) {
    float* As = gsm + buf * SF;   // [BK][BM]
    float* Bs = As + kGemmBK * BM;  // [BK][BN]
    const int k0 = kt * kGemmBK;
    for (int idx = tid; idx < kGemmBK * BM / 4; idx += kGemmThreads) {
      const int kk = idx / (BM / 4), c4 = (idx % (BM / 4)) * 4;
      const int k = k0 + kk;
      const bool va = k < Kw && o0 + c4 < ldw;
      cp_async16(As + kk * BM + c4, va ? Wt + (long long)k * ldw + o0 + c4 : Wt, va);
    }
#pragma unroll
    for (int r = 0; r < kGemmBK * BN / 4 / kGemmThreads; ++r) {
      const int idx = tid + r * kGemmThreads;
      const int kk = idx / (BN / 4), c4 = (idx % (BN / 4)) * 4;
      cp_async16(Bs + kk * BN + c4, X + (long long)(k0 + kk) * ldx + c0 + c4, true);
    }
  };

  // accumulators as packed column pairs (FFMA2): acc2[a][q] = columns 2q, 2q+1
  unsigned long long acc2[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc2[a][q] = 0ull;

  const int KT = K / kGemmBK;
#pragma unroll
  for (int s = 0; s < kGemmStages - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<kGemmStages - 2>();
    __syncthreads();  // stage kt visible; stage kt-1's buffer free for the refill
    if (kt + kGemmStages - 1 < KT) load_stage(kt + kGemmStages - 1, (kt + kGemmStages - 1) % kGemmStages);
    cp_async_commit();
    const float* As = gsm + (kt % kGemmStages) * SF;
    const float* Bs = As + kGemmBK * BM;
    auto kstep = [&](int kk) {
      if constexpr (OPT == 8) {
        const float4 a0 = *reinterpret_cast<const float4*>(As + kk * BM + ob);
        const float4 a1 = *reinterpret_cast<const float4*>(As + kk * BM + ob + 16);
        const float4 b0 = *reinterpret_cast<const float4*>(Bs + kk * BN + cb);
        const float4 b1 = *reinterpret_cast<const float4*>(Bs + kk * BN + cb + 32);
        const float w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const unsigned long long x2[4] = {f32x2_pack(b0.x, b0.y), f32x2_pack(b0.z, b0.w),
                                          f32x2_pack(b1.x, b1.y), f32x2_pack(b1.z, b1.w)};
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int q = 0; q < 4; ++q) ffma2_bcast(acc2[a][q], w[a], x2[q]);
      } else {
        const float4 b0 = *reinterpret_cast<const float4*>(Bs + kk * BN + cb);
        const float4 b1 = *reinterpret_cast<const float4*>(Bs + kk * BN + cb + 32);
        const unsigned long long x2[4] = {f32x2_pack(b0.x, b0.y), f32x2_pack(b0.z, b0.w),
                                          f32x2_pack(b1.x, b1.y), f32x2_pack(b1.z, b1.w)};
        float w[OPT];
#pragma unroll
        for (int a = 0; a < OPT; ++a) w[a] = As[kk * BM + oy * OPT + a];
#pragma unroll
        for (int a = 0; a < OPT; ++a)
#pragma unroll
          for (int q = 0; q < 4; ++q) ffma2_bcast(acc2[a][q], w[a], x2[q]);
      }
    };
    const int kk_end = Kw - kt * kGemmBK;  // the weight rows that exist
    if (kk_end >= kGemmBK) {
#pragma unroll
      for (int kk = 0; kk < kGemmBK; ++kk) kstep(kk);
    } else {
      // zero-padded K rows (the first layer's K = 3E+3 -> multiple of 16) are
      // skipped: their weights and inputs are 0, and adding fmaf(0, x, acc)
      // is the identity (acc is never -0), so the bits are unchanged
#pragma unroll 1
      for (int kk = 0; kk < kk_end; ++kk) kstep(kk);
    }
  }
  cp_async_wait<0>();
  float acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 v = f32x2_unpack(acc2[a][q]);
      acc[a][2 * q] = v.x;
      acc[a][2 * q + 1] = v.y;
    }

  // epilogue: + bias (then ReLU); hidden -> Y[o][col], last -> raw[col][o]
#pragma unroll
  for (int a = 0; a < OPT; ++a) {
    const int o = (OPT == 8) ? o0 + ob + (a < 4 ? a : 12 + a) : o0 + oy * OPT + a;
    if (o >= out) {  // hidden: rows out..roundup16(out) are the next layer's K padding
      if (!LAST && o < ((out + 15) & ~15))
#pragma unroll
        for (int h = 0; h < 2; ++h)
          *reinterpret_cast<float4*>(Y + (long long)o * ldy + c0 + cb + h * 32) =
              make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    const float bo = bias[o];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = c0 + cb + h * 32;
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float z = acc[a][h * 4 + j] + bo;
        v[j] = LAST ? z : (z > 0.f ? z : 0.f);
      }
      if (LAST) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c + j < ncols) raw[(long long)(c + j) * out + o] = v[j];
      } else {
        *reinterpret_cast<float4*>(Y + (long long)o * ldy + c) = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
  }
}

}  // namespace cyr

// Worth it when some layer is wider than one 256-output panel (the fused
// kernel's tiles shrink to 8 columns) and the batch fills the machine with
// 128-column tiles; single-panel actors (cfg2) only from 65,536 columns on,
// where the GEMM's 70 % FMA-pipe rate beats the fused kernel's 56 % despite
// the activation round trips (cfg2 Mode-T tree 3.49 -> 3.21 ms).
// CYR_ACTOR_GEMM=wide restricts the path to multi-panel actors, =0
// disables it (A/B).
bool cyr_gemm_path_applies(int precision, const cyr::ActorDesc& desc, long long ncols) {
  static const int mode = [] {
    const char* e = getenv("CYR_ACTOR_GEMM");
    return e == nullptr ? 2 : (e[0] == '0' ? 0 : (e[0] == 'w' ? 1 : 2));
  }();
  if (mode == 0 || precision != CYR_FP32 || ncols < 2048) return false;
  for (int l = 0; l < desc.n_layers; ++l)
    if (desc.layer[l].out_pad > 256) return true;
  return mode == 2 && ncols >= 65536;
}

// workspace: two activation buffers of max_width (rounded to 16) x
// roundup(ncols, 512) floats
size_t cyr_gemm_workspace_bytes(const cyr::ActorDesc& desc, long long ncols) {
  const long long ldx = cyr::gemm_ldx(ncols);
  int rows = 0;
  for (int l = 0; l < desc.n_layers; ++l)
    rows = std::max(rows, std::max((desc.layer[l].in + 15) / 16 * 16, desc.layer[l].out));
  return 2ull * (size_t)rows * (size_t)ldx * sizeof(float);
}

namespace {
template <int BM, int BN, bool LAST, int OPT = 8>
int launch_layer(const float* Wt, int ldw, int Kw, const float* bias, const float* X, int ldx, int K,
                 int out, float* Y, float* raw, int ncols, cudaStream_t stream) {
  using namespace cyr;
  constexpr size_t smem = (size_t)kGemmStages * stage_floats<BM, BN>() * sizeof(float);
  auto kern = sgemm_layer_kernel<BM, BN, LAST, OPT>;
  static AttrCache configured;
  if (!ensure_func_attr(configured, (int)smem, [&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem) == cudaSuccess;
      }))
    return CYR_CUDA_ERROR;
  const dim3 grid((unsigned)((ncols + BN - 1) / BN), (unsigned)((out + BM - 1) / BM));
  kern<<<grid, kGemmThreads, smem, stream>>>(Wt, ldw, Kw, bias, X, ldx, K, out, Y, ldx, raw, ncols);
  return CYR_OK;
}
}  // namespace

int cyr_launch_actor_gemm(const cyr::ActorLaunch& p, void* workspace, cudaStream_t stream) {
  using namespace cyr;
  const long long ncols = p.ncols;
  if (ncols <= 0) return CYR_OK;
  const int ldx = gemm_ldx(ncols);
  const size_t half = cyr_gemm_workspace_bytes(p.desc, ncols) / 2;
  float* buf[2] = {static_cast<float*>(workspace),
                   reinterpret_cast<float*>(static_cast<unsigned char*>(workspace) + half)};
  const float* blob = static_cast<const float*>(p.blob);
  const int k0pad = (p.desc.layer[0].in + 15) / 16 * 16;
  {
    const long long n = (long long)k0pad * ldx;
    const int blocks = (int)std::min<long long>((n + 255) / 256, 148ll * 16);
    if (p.x == nullptr && p.kcol == nullptr && p.cap >= 1) {
      const long long groups = (ldx + p.cap - 1) / p.cap;
      const int gblocks = (int)std::min<long long>((groups + 255) / 256, 148ll * 16);
      gemm_features_group_kernel<<<gblocks, 256, 0, stream>>>(p, buf[0], ldx, k0pad);
    } else {
      gemm_features_kernel<<<blocks, 256, 0, stream>>>(p, buf[0], ldx, k0pad);
    }
  }
  int cur = 0;
  for (int l = 0; l < p.desc.n_layers; ++l) {
    const LayerDesc& L = p.desc.layer[l];
    const bool last = l == p.desc.n_layers - 1;
    const int K = (L.in + 15) / 16 * 16;
    const float* W = blob + L.w_off;
    const float* b = blob + L.b_off;
    int rc;
    if (last && L.out <= kHeadBM) {
      auto head = [&](auto opt) {
        return launch_layer<kHeadBM, kHeadBN, true, decltype(opt)::value>(
            W, L.out_pad, L.in, b, buf[cur], ldx, K, L.out, nullptr, static_cast<float*>(p.raw),
            p.ncols, stream);
      };
      switch ((L.out + 3) / 4) {  // outputs per thread, no padded rows
        case 1: rc = head(std::integral_constant<int, 1>{}); break;
        case 2: rc = head(std::integral_constant<int, 2>{}); break;
        case 3: rc = head(std::integral_constant<int, 3>{}); break;
        case 4: rc = head(std::integral_constant<int, 4>{}); break;
        case 5: rc = head(std::integral_constant<int, 5>{}); break;
        case 6: rc = head(std::integral_constant<int, 6>{}); break;
        case 7: rc = head(std::integral_constant<int, 7>{}); break;
        default: rc = head(std::integral_constant<int, 8>{}); break;
      }
    } else if (last) {
      rc = launch_layer<kGemmBM, kGemmBN, true>(W, L.out_pad, L.in, b, buf[cur], ldx, K, L.out,
                                                nullptr, static_cast<float*>(p.raw), p.ncols, stream);
    } else {
      rc = launch_layer<kGemmBM, kGemmBN, false>(W, L.out_pad, L.in, b, buf[cur], ldx, K, L.out,
                                                 buf[cur ^ 1], nullptr, p.ncols, stream);
    }
    if (rc != CYR_OK) return rc;
    cur ^= 1;
  }
  return cudaPeekAtLastError() == cudaSuccess ? CYR_OK : CYR_CUDA_ERROR;
}
