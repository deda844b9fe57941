// Pure-write HBM patterns on B200: what ceiling does each store mechanism
// reach for a 3.2 GB output (the K1 tree's per-step bytes)?
//   A: st.global.v4 from registers, grid-stride, coalesced (torch fill-like)
//   B: TMA bulk store (cp.async.bulk.global.shared) of NP*160 B items from a
//      double-buffered shared-memory stage, persistent 2 CTAs/SM (K1's scheme)
//   C: like B but 4 stage buffers / 4 stores in flight per CTA
//   D: st.global.v4 of the same item layout written from smem-staged data
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wp write_patterns.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__global__ void k_a(uint4* out, long long n16) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = make_uint4((unsigned)i, 1, 2, 3);
}

template <int NST>
__global__ void k_b(unsigned char* out, int items, int item_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  int it = 0;
  for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
    unsigned char* st = sm + (size_t)(it % NST) * item_bytes;
    if (threadIdx.x == 0) bulk_wait_read<NST - 1>();
    __syncthreads();
    uint4* s4 = reinterpret_cast<uint4*>(st);
    for (int c = threadIdx.x; c < item_bytes / 16; c += blockDim.x) s4[c] = make_uint4(w, c, 0, 1);
    fence_proxy();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(out + (long long)w * item_bytes, st, item_bytes);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

__global__ void k_d(unsigned char* out, int items, int item_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    uint4* s4 = reinterpret_cast<uint4*>(sm);
    __syncthreads();
    for (int c = threadIdx.x; c < item_bytes / 16; c += blockDim.x) s4[c] = make_uint4(w, c, 0, 1);
    __syncthreads();
    uint4* o = reinterpret_cast<uint4*>(out + (long long)w * item_bytes);
    for (int c = threadIdx.x; c < item_bytes / 16; c += blockDim.x) o[c] = s4[c];
  }
}

int main() {
  const long long bytes = 3200163840ll;
  unsigned char* buf;
  cudaMalloc(&buf, bytes + (1 << 20));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-48s %8.3f ms  %6.0f GB/s  (%s)\n", name, best, bytes / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  timeit("A st.global.v4 grid-stride (sms*8 x 256)", [&] {
    k_a<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(buf), bytes / 16);
  });
  for (int np : {64, 128, 256}) {
    const int item = np * 160, items = (int)(bytes / item);
    for (int per : {1, 2, 3, 4}) {
      const size_t sm2 = 2ull * item, sm4 = 4ull * item;
      if (per * (sm2 + 2048) <= 228 * 1024) {
        cudaFuncSetAttribute(k_b<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
        char nm[96];
        snprintf(nm, sizeof nm, "B TMA item %d B, 2 stages, %d CTA/SM", item, per);
        timeit(nm, [&] { k_b<2><<<sms * per, 256, sm2>>>(buf, items, item); });
      }
      if (per * (sm4 + 2048) <= 228 * 1024) {
        cudaFuncSetAttribute(k_b<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
        char nm[96];
        snprintf(nm, sizeof nm, "C TMA item %d B, 4 stages, %d CTA/SM", item, per);
        timeit(nm, [&] { k_b<4><<<sms * per, 256, sm4>>>(buf, items, item); });
      }
    }
    cudaFuncSetAttribute(k_d, cudaFuncAttributeMaxDynamicSharedMemorySize, item);
    char nm[96];
    snprintf(nm, sizeof nm, "D smem->st.global.v4 item %d B, 2 CTA/SM", item);
    timeit(nm, [&] { k_d<<<sms * 2, 256, item>>>(buf, items, item); });
    snprintf(nm, sizeof nm, "D smem->st.global.v4 item %d B, 4 CTA/SM", item);
    if (4 * (item + 2048) <= 228 * 1024) timeit(nm, [&] { k_d<<<sms * 4, 256, item>>>(buf, items, item); });
  }
  return 0;
}
