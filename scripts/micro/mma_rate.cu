// tcgen05.mma dispatch rate on B200 for the narrow-MLP shapes (M = 128,
// K = 16 per instruction, bf16): cycles per instruction vs N, SS vs TS (A in
// TMEM), one accumulator vs rotating accumulators, one CTA alone vs one CTA
// per SM.  Operands are zero (the rate does not depend on values).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT;\n\t}" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}

constexpr int kIters = 256;

__global__ void __launch_bounds__(128) mma_rate(long long* out, int variant) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  uint32_t phase = 0;
  if (warp == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 16 * 1024);
    int slot = 0;
    // configs: N in {32, 64, 128, 256} x {SS, TS} x {1 acc, 4 rotating accs (N <= 64)}
    for (int n = 32; n <= 256; n *= 2)
      for (int ts = 0; ts < 2; ++ts)
        for (int rot = 0; rot < 2; ++rot) {
          if (rot && n > 64) { if (threadIdx.x == 0) out[blockIdx.x * 32 + slot] = -1; ++slot; continue; }
          const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);
          __syncwarp();
          const long long c0 = clock64();
          if (variant == 1) {  // descriptors hoisted: the same A/B every MMA, unrolled by 8
            const uint64_t ad = desc_sw128(a), bd = desc_sw128(b);
            for (int k = 0; k < kIters; k += 8) {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                if (ts) mma_ts(tmem, tmem + 256u, bd, id, 1);
                else mma_ss(tmem, ad, bd, id, 1);
              }
            }
          } else if (variant == 2) {  // M = 64
            const uint32_t id64 = (id & ~(0x1fu << 24)) | ((uint32_t)(64 >> 4) << 24);
            const uint64_t ad = desc_sw128(a), bd = desc_sw128(b);
            for (int k = 0; k < kIters; k += 8) {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                if (ts) mma_ts(tmem, tmem + 256u, bd, id64, 1);
                else mma_ss(tmem, ad, bd, id64, 1);
              }
            }
          } else if (variant == 3) {  // 8 MMAs in one asm block: no per-MMA issue overhead
            const uint64_t ad = desc_sw128(a), bd = desc_sw128(b);
            for (int k = 0; k < kIters; k += 8) {
              if (ts)
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}"
                    ::"r"(tmem), "r"(tmem + 256u), "l"(bd), "r"(id) : "memory");
              else
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}"
                    ::"r"(tmem), "l"(ad), "l"(bd), "r"(id) : "memory");
            }
          } else if (variant == 4) {  // 4 MMAs per asm block, distinct per-MMA operands (real use)
            for (int k = 0; k < kIters; k += 4) {
              uint64_t bd[4];
              uint32_t at[4];
              uint64_t ad[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int kk = k + u;
                bd[u] = desc_sw128(b + (uint32_t)((kk >> 2) & 1) * (uint32_t)n * 128u + (uint32_t)(kk & 3) * 32u);
                at[u] = tmem + 256u + (uint32_t)((kk & 15) * 8);
                ad[u] = desc_sw128(a + (uint32_t)(kk & 3) * 32u);
              }
              if (ts)
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %9, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %6, %9, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %7, %9, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %8, %9, 1;\n\t}"
                    ::"r"(tmem), "r"(at[0]), "r"(at[1]), "r"(at[2]), "r"(at[3]),
                      "l"(bd[0]), "l"(bd[1]), "l"(bd[2]), "l"(bd[3]), "r"(id) : "memory");
              else
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %5, %9, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %6, %9, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %7, %9, 1;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %8, %9, 1;\n\t}"
                    ::"r"(tmem), "l"(ad[0]), "l"(ad[1]), "l"(ad[2]), "l"(ad[3]),
                      "l"(bd[0]), "l"(bd[1]), "l"(bd[2]), "l"(bd[3]), "r"(id) : "memory");
            }
          } else if (variant == 5) {  // per-MMA asm, NO elect (whole warp executes; uniform op)
            for (int k = 0; k < kIters; ++k) {
              const uint64_t bd = desc_sw128(b + (uint32_t)((k >> 2) & 1) * (uint32_t)n * 128u + (uint32_t)(k & 3) * 32u);
              if (ts)
                asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;"
                             ::"r"(tmem), "r"(tmem + 256u + (uint32_t)((k & 15) * 8)), "l"(bd), "r"(id) : "memory");
              else
                asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;"
                             ::"r"(tmem), "l"(desc_sw128(a + (uint32_t)(k & 3) * 32u)), "l"(bd), "r"(id) : "memory");
            }
          } else if (variant == 6) {  // 16 MMAs per asm, operands computed inside the asm
            for (int k = 0; k < kIters; k += 16) {
              const uint64_t bd = desc_sw128(b + (uint32_t)((k >> 4) & 1) * (uint32_t)n * 128u);
              asm volatile(
                    "{\n\t.reg .pred e;\n\t.reg .b32 ta;\n\t.reg .b64 bd;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "add.u32 ta, %1, 0;\n\tadd.u64 bd, %2, 0;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 8;\n\tadd.u64 bd, %2, 2;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 16;\n\tadd.u64 bd, %2, 4;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 24;\n\tadd.u64 bd, %2, 6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 32;\n\tadd.u64 bd, %2, 0;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 40;\n\tadd.u64 bd, %2, 2;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 48;\n\tadd.u64 bd, %2, 4;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 56;\n\tadd.u64 bd, %2, 6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 64;\n\tadd.u64 bd, %2, 0;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 72;\n\tadd.u64 bd, %2, 2;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 80;\n\tadd.u64 bd, %2, 4;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 88;\n\tadd.u64 bd, %2, 6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 96;\n\tadd.u64 bd, %2, 0;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 104;\n\tadd.u64 bd, %2, 2;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 112;\n\tadd.u64 bd, %2, 4;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 120;\n\tadd.u64 bd, %2, 6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "}"
                    ::"r"(tmem), "r"(tmem + 256u), "l"(bd), "r"(id) : "memory");
            }
          } else if (variant == 7) {  // 4 MMAs per asm (one K tile), in-asm operand arithmetic
            for (int k = 0; k < kIters; k += 4) {
              const uint64_t bd = desc_sw128(b + (uint32_t)((k >> 2) & 1) * (uint32_t)n * 128u);
              asm volatile(
                    "{\n\t.reg .pred e;\n\t.reg .b32 ta;\n\t.reg .b64 bd;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
                    "add.u32 ta, %1, 8;\n\tadd.u64 bd, %2, 2;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 16;\n\tadd.u64 bd, %2, 4;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "add.u32 ta, %1, 24;\n\tadd.u64 bd, %2, 6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
                    "}"
                    ::"r"(tmem), "r"(tmem + 256u + (uint32_t)((k & 15) * 8)), "l"(bd), "r"(id) : "memory");
            }
          } else
          for (int k = 0; k < kIters; ++k) {
            const uint32_t dcol = rot ? (uint32_t)((k & 3) * 64) : 0u;
            const uint64_t bd = desc_sw128(b + (uint32_t)((k >> 2) & 1) * (uint32_t)n * 128u +
                                           (uint32_t)(k & 3) * 32u);
            if (ts)
              mma_ts(tmem + dcol, tmem + 256u + (uint32_t)((k & 15) * 8), bd, id, (rot ? k >= 4 : k > 0));
            else
              mma_ss(tmem + dcol, desc_sw128(a + (uint32_t)(k & 3) * 32u), bd, id, (rot ? k >= 4 : k > 0));
          }
          const long long c1 = clock64();
          commit(&bar);
          mbar_wait(&bar, phase);
          phase ^= 1;
          const long long c2 = clock64();
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (threadIdx.x == 0) {
            out[blockIdx.x * 32 + slot] = c2 - c0;
            out[blockIdx.x * 32 + 16 + slot] = c1 - c0;
          }
          ++slot;
        }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// In-context rate: TS N=256 MMAs in groups of 4 (one asm), B cycling over
// `btiles` distinct 32 KB K tiles, while `spin` other warps poll an mbarrier
// (the fused MLP's idle epilogue warps do exactly that during MMA2).
__global__ void __launch_bounds__(512) mma_ctx(long long* out, int btiles, int spin, int n, int busy, uint32_t dcol, uint32_t acol, int rnd) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 128 * 1024 / 16; i += blockDim.x) {
    uint32_t h = rnd ? (uint32_t)i * 2654435761u : 0u;
    // bf16 pairs in [-1, 1): sign/exponent 0x3f.. / 0xbf.., random mantissa
    const uint32_t w = rnd ? ((h & 0x007f007fu) | 0x3f003f00u | (h & 0x80008000u)) : 0u;
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(w, w ^ 0x00550055u, w ^ 0x002a002au, w ^ 0x00110011u);
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&done, 1); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (rnd && warp < 4) {  // random bf16 pairs into every TMEM column (lane quarter = warp)
    for (int c = 0; c < 512; ++c) {
      uint32_t h = (uint32_t)(c * 131 + threadIdx.x) * 2654435761u;
      const uint32_t w = (h & 0x007f007fu) | 0x3f003f00u | (h & 0x80008000u);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c), "r"(w) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    const uint32_t b = smem_u32(sm);
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
                        ((uint32_t)(128 >> 4) << 24);
    __syncwarp();
    // let the busy warps start
    const long long cs = clock64();
    while (clock64() - cs < 2000) {}
    const long long c0 = clock64();
    for (int k = 0; k < kIters; k += 4) {
      const uint64_t bd = desc_sw128(b + (uint32_t)((k >> 2) % btiles) * 32768u);
      asm volatile(
          "{\n\t.reg .pred e;\n\t.reg .b32 ta;\n\t.reg .b64 bd;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"
          "add.u32 ta, %1, 8;\n\tadd.u64 bd, %2, 2;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
          "add.u32 ta, %1, 16;\n\tadd.u64 bd, %2, 4;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
          "add.u32 ta, %1, 24;\n\tadd.u64 bd, %2, 6;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t}"
          ::"r"(tmem + dcol), "r"(tmem + acol + (uint32_t)((k & 15) * 8)), "l"(bd), "r"(id) : "memory");
    }
    commit(&bar);
    mbar_wait(&bar, 0);
    const long long c2 = clock64();
    if (threadIdx.x == 0) {
      out[blockIdx.x] = c2 - c0;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done)) : "memory");
    }
  } else if (warp <= spin) {
    mbar_wait(&done, 0);
  } else if (warp <= spin + busy) {  // FMA + shared-store heavy (a feature builder's mix)
    float x = threadIdx.x * 1e-3f, y = 1.0001f;
    uint32_t sp = smem_u32(sm + 64 * 1024) + (threadIdx.x & 127) * 4;
    for (int it = 0; it < 4000; ++it) {
#pragma unroll
      for (int u = 0; u < 8; ++u) x = fmaf(x, y, 0.5f);
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(sp), "f"(x) : "memory");
    }
    if (x == 12345.f) out[0] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// The fused MLP's exact MMA2 -> MMA3 sequence: 16 x (N = 256, A cols 256..)
// into D cols 0..255, commit + wait, then 16 x (N = 32, A cols 384..) into
// D cols 256..287, one asm per K tile of 4; clocks per group of 4.
__device__ __forceinline__ void ts_x4(uint32_t d, uint32_t a, uint64_t bd, uint32_t id, int acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 ta;\n\t.reg .b64 bd;\n\t"
      "setp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "add.u32 ta, %1, 8;\n\tadd.u64 bd, %2, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
      "add.u32 ta, %1, 16;\n\tadd.u64 bd, %2, 4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t"
      "add.u32 ta, %1, 24;\n\tadd.u64 bd, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %3, 1;\n\t}"
      ::"r"(d), "r"(a), "l"(bd), "r"(id), "r"(acc) : "memory");
}
__global__ void __launch_bounds__(128) mma_seq(long long* out, int with_mma2, int acc0, int write_a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (write_a) {  // all 4 warps: fresh A3 (cols 384..511) via tcgen05.st right before MMA3
    for (int c = 0; c < 128; c += 16) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) r[j] = 0x3f803f80u ^ (uint32_t)(threadIdx.x * 16 + j + c);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tmem_base + ((uint32_t)(warp * 32) << 16) + 384u + (uint32_t)c),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (warp == 0) {
    const uint32_t w2 = smem_u32(sm), w3 = smem_u32(sm + 128 * 1024);
    const uint32_t id2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | (8u << 24);
    const uint32_t id3 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(32 >> 3) << 17) | (8u << 24);
    long long c[8];
    uint32_t ph = 0;
    for (int rep = 0; rep < 3; ++rep) {
      if (with_mma2) {
        for (int ks = 0; ks < 16; ks += 4)
          ts_x4(0u, 256u + ks * 8, desc_sw128(w2 + (ks >> 2) * 256 * 128), id2, ks > 0);
        commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      c[0] = clock64();
      for (int ks = 0; ks < 16; ks += 4) {
        ts_x4(256u, 384u + ks * 8, desc_sw128(w3 + (ks >> 2) * 32 * 128), id3, acc0 ? 1 : ks > 0);
        c[1 + ks / 4] = clock64();
      }
      commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      c[5] = clock64();
    }
    if (threadIdx.x == 0)
      for (int j = 0; j < 5; ++j) out[j] = c[j + 1] - c[0];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

int main() {
  long long* d;
  long long h[148 * 32];
  cudaMalloc(&d, sizeof(h));
  const int smem = 97 * 1024 + 1024;
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int variant = 7; variant < 7; ++variant)
  for (int grid : {1, 148}) {
    for (int rep = 0; rep < 2; ++rep) {
      mma_rate<<<grid, 128, smem>>>(d, variant);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int slot = 0;
    for (int n = 32; n <= 256; n *= 2)
      for (int ts = 0; ts < 2; ++ts)
        for (int rot = 0; rot < 2; ++rot, ++slot) {
          if (h[slot] < 0) continue;
          printf("v%d grid %3d N=%3d %s %s: %6.1f cycles/mma (issue %6.1f), ideal %d\n", variant, grid, n,
                 ts ? "TS" : "SS", rot ? "4 accs" : "1 acc ", (double)h[slot] / kIters,
                 (double)h[16 + slot] / kIters, 128 * n / 256);
        }
  }
  {
    const int smem2 = 129 * 1024;
    cudaFuncSetAttribute(mma_ctx, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    const uint32_t cols[][2] = {{0, 256}, {256, 384}};
    for (int rnd : {0})
    for (int n : {32})
      for (auto& dc : cols) {
          if (dc[0] + n > 512 || (dc[0] < dc[1] + 128 && dc[1] < dc[0] + n)) continue;
          mma_ctx<<<148, 512, smem2>>>(d, 1, 0, n, 0, dc[0], dc[1], rnd);
          mma_ctx<<<148, 512, smem2>>>(d, 1, 0, n, 0, dc[0], dc[1], rnd);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
          printf("ctx %s TS N=%d x4 in-asm: D col %u, A cols %u..%u: %6.1f cycles/mma\n", rnd ? "random" : "zeros ", n, dc[0],
                 dc[1], dc[1] + 127, (double)h[0] / kIters);
      }
  }
  {
    const int smem3 = 161 * 1024 + 1024;
    cudaFuncSetAttribute(mma_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    for (int wa : {0, 1})
    for (int w2 : {0, 1})
      for (int acc0 : {0}) {
        mma_seq<<<1, 128, smem3>>>(d, w2, acc0, wa);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 5 * sizeof(long long), cudaMemcpyDeviceToHost);
        printf("seq: A3 written by tcgen05.st %d, MMA2 first %d, first MMA3 acc %d: groups %lld %lld %lld %lld, done %lld\n", wa, w2,
               acc0, h[0], h[1], h[2], h[3], h[4]);
        (void)wa;
      }
  }
  return 0;
}
