// tcgen05.mma throughput probe (dev tool): cycles per 128 x N x 16 bf16 MMA issued
// back to back by one thread, per SM, for several N and shared-memory layouts.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2307_08771_b200/csrc
//        tools/mma_probe.cu -o gpurun_out/mma_probe
#include <cstdio>

#include "ub_common.cuh"

using namespace ub;

UB_DEVI uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(layout & 7u) << 61;
  return d;
}

// mode 0: SW128 A and B (K advanced by 32 B inside the atom)
// mode 1: no-swizzle A and B, aligned (LBO 2048 / 4096)
// mode 2: no-swizzle A with LBO 16 (overlapping, shifted-row trick), B no-swizzle
// commit_every: commit + wait after this many MMAs (0 = only at the end)
__global__ void __launch_bounds__(128, 1) probe_mma(int n, int mode, int iters, int commit_every,
                                                    unsigned long long* out, int shift = 48) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  uint8_t* sA = base;          // 16 KB
  uint8_t* sB = base + 16384;  // 32 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = slot;
  if (mode == 5 && threadIdx.x < 32) {  // whole warp, elect.sync inside the asm
    const uint32_t idesc = make_idesc_bf16(128, n);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (commit_every == 1) {  // no-swizzle planes: A rows 16 B apart, K core matrices 4 KB apart
        ad[k] = sdesc(a0 + k * shift, 4096, 128, 0);
        bd[k] = sdesc(b0, n * 16, 128, 0);
      } else if (commit_every == 2) {  // SW64 A (64-byte rows, row shifts of k), SW128 B
        ad[k] = sdesc(a0 + (k & 1) * 32 + k * 64, 16, 512, 4);
        bd[k] = sdesc(b0 + (k & 1) * 32, 16, 1024, 2);
      } else {
        ad[k] = sdesc(a0 + k * 32, 16, 1024, 2);
        bd[k] = sdesc(b0 + k * 32, 16, 1024, 2);
      }
    }
    __syncwarp();
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "elect.sync _|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
            "l"(ad[k]), "l"(bd[k]), "r"(idesc)
            : "memory");
    }
    if (threadIdx.x == 0) {
      umma_commit(&bar);
      mbar_wait(&bar, 0);
    }
    __syncwarp();
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  } else if (mode < 5 && threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(128, n);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    uint32_t ph = 0;
    const long long t0 = clock64();
    if (mode >= 3) {  // precomputed descriptors, 4 MMAs unrolled per iteration
      uint64_t ad[4], bd[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ad[k] = sdesc(a0 + k * 32, 16, 1024, 2);
        bd[k] = sdesc(b0 + k * 32, 16, 1024, 2);
      }
      for (int i = 0; i < iters; i += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_bf16(d, ad[k], bd[k], idesc, 1u);
        if (mode == 4 && commit_every && (i + 4) % commit_every == 0) {
          umma_commit(&bar);
          mbar_wait(&bar, ph);
          ph ^= 1;
        }
      }
      iters = 0;
    }
    for (int i = 0; i < iters; ++i) {
      const int k = i & 3;
      uint64_t ad, bd;
      if (mode == 0) {
        ad = sdesc(a0 + k * 32, 16, 1024, 2);
        bd = sdesc(b0 + k * 32, 16, 1024, 2);
      } else if (mode == 1) {
        ad = sdesc(a0, 2048, 128, 0);
        bd = sdesc(b0, n * 16, 128, 0);
      } else {
        ad = sdesc(a0 + k * 16, 16, 128, 0);
        bd = sdesc(b0, n * 16, 128, 0);
      }
      umma_bf16(d, ad, bd, idesc, 1u);
      if (commit_every && (i + 1) % commit_every == 0) {
        umma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, ph);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(d, 256);
  }
}

int main() {
  unsigned long long* dout;
  cudaMalloc(&dout, 8);
  cudaFuncSetAttribute(probe_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4096;
  const char* names[6] = {"sw128", "noswz", "noswz-lbo16", "sw128-pre", "sw128-pre-c", "warp-elect"};
  for (int mode = 5; mode < 6; ++mode) {
    for (int n : {32, 64, 128}) {
      for (int sh : {-1, -2, 0, 48}) {
        const int ce = sh == -1 ? 0 : (sh == -2 ? 2 : 1);
        for (int grid : {148}) {
          probe_mma<<<grid, 128, 64 * 1024>>>(n, mode, iters, ce, dout, sh);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          unsigned long long cyc = 0;
          cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost);
            printf("shift %4d ", sh);
          printf("%-12s N=%3d planes=%d grid=%3d: %6.1f cyc/MMA (ideal %5.1f)\n", names[mode], n, ce, grid,
                 double(cyc) / iters, 128.0 * n / 256.0);
        }
      }
    }
  }
  return 0;
}
