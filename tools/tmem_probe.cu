// TMEM -> register read throughput probe (dev tool): W warps (lane quarter = warp % 4) each
// issue tcgen05.ld.32x32b.x32 (+ wait) in a loop; optionally one warp keeps the tensor core
// busy with MMAs into other columns at the same time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2307_08771_b200/csrc
//        tools/tmem_probe.cu -o tools/tmem_probe_bin
#include <cstdio>

#include "ub_common.cuh"

using namespace ub;

UB_DEVI void ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
      " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
UB_DEVI void ld_16x128b_x16(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x128b.x16.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
      " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

__global__ void __launch_bounds__(640, 1) probe(int ldw, int iters, int with_mma, int batch, int shape, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    stop = 0;
  }
  for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 19) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t0 = slot;
  if (warp < ldw) {
    const int q = warp & 3;
    long long c0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
      uint32_t v0[32], v1[32];
      const uint32_t ta = t0 + (static_cast<uint32_t>(q * 32) << 16) + (((warp >> 2) * 64) & 255);
      if (shape == 0) tmem_ld32(ta, v0);
      else if (shape == 1) ld_16x256b_x8(ta, v0);
      else ld_16x128b_x16(ta, v0);
      if (batch > 1) {
        if (shape == 0) tmem_ld32(ta + 32, v1);
        else if (shape == 1) ld_16x256b_x8(ta + 32, v1);
        else ld_16x128b_x16(ta + 32, v1);
      }
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += v0[k] ^ (batch > 1 ? v1[k] : 0u);
    }
    long long c1 = clock64();
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[warp] = c1 - c0;
    if (acc == 12345) out[40] = acc;
    __syncthreads();
  } else if (warp == 18 && with_mma) {
    const uint32_t idesc = make_idesc_bf16(128, 256);
    const uint64_t ad = make_sdesc(smem_u32(base), 1024, 2), bd = make_sdesc(smem_u32(base + 16384), 1024, 2);
    int n = 0;
    while (!stop && n < 100000) {
      for (int k = 0; k < 16; ++k) umma_bf16_warp(t0 + 256, ad, bd, idesc, 1u);
      n += 16;
      umma_commit_warp(&bar);
      mbar_wait(&bar, ((n / 16) - 1) & 1);
    }
    __syncthreads();
  } else {
    __syncthreads();
  }
  if (threadIdx.x == 0) stop = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 19) {
    tc_fence_after();
    tmem_dealloc(t0, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 2000;
  const char* names[3] = {"32x32b.x32", "16x256b.x8", "16x128b.x16"};
  for (int shape = 0; shape < 3; ++shape)
  for (int mma = 0; mma < 1; ++mma)
    for (int ldw : {1, 4, 8, 16})
      for (int batch : {1, 2}) {
        probe<<<148, 640, 64 * 1024>>>(ldw, iters, mma, batch, shape, d);
        if (cudaDeviceSynchronize() != cudaSuccess) {
          printf("error\n");
          return 1;
        }
        unsigned long long c[64];
        cudaMemcpy(c, d, 64 * 8, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int w = 0; w < ldw; ++w) mx = c[w] > mx ? c[w] : mx;
        const double bytes = double(ldw) * iters * batch * 32 * 32 * 4;
        printf("%s mma=%d warps=%2d batch=%d: %7.1f cycles/iter/warp, %6.1f B/clk/SM\n", names[shape], mma, ldw, batch,
               double(mx) / iters, bytes / double(mx));
      }
  return 0;
}
