// TMA throughput probe (dev tool): how many bytes/s does one SM's TMA unit move
// as a function of the box row size?  148 persistent CTAs stream boxes of
// {inner_elems bf16, rows} from a 1 GiB tensor into a 4-stage smem ring.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2307_08771_b200/csrc
//        tools/tma_probe.cu -o gpurun_out/tma_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ub_common.cuh"

using namespace ub;

__global__ void __launch_bounds__(128, 1) probe_load(const __grid_constant__ CUtensorMap tm, int rows_total, int box_rows,
                                                      int box_bytes, int iters, unsigned long long* sink, int S) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * box_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nblk = rows_total / box_rows;
    int b = blockIdx.x;
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&bar[s], ((i - S) / S) & 1);
      mbar_arrive_expect_tx(&bar[s], box_bytes);
      tma_load_2d(&tm, &bar[s], smem + s * box_bytes, 0, (b % nblk) * box_rows);
      b += gridDim.x;
    }
    for (int i = iters; i < iters + S; ++i) {
      const int s = i % S;
      mbar_wait(&bar[s], ((i - S) / S) & 1);
    }
    sink[blockIdx.x] = smem[5];
  }
}

// LSU streaming: each warp copies rows of `row_bytes` (16 B per lane-slot) with cp.async into smem.
template <int DEPTH>
__global__ void __launch_bounds__(512, 1) probe_cpasync(const uint8_t* src, long long rows_total, int pitch, int row_bytes,
                                                         int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int per_row = row_bytes / 16;
  const int rows_per_iter = blockDim.x / per_row;  // one 16-B piece per thread per iteration
  const int tid = threadIdx.x;
  long long row = (long long)blockIdx.x * rows_per_iter;
  const long long stride = (long long)gridDim.x * rows_per_iter;
  for (int i = 0; i < iters; ++i) {
    const long long r = (row + tid / per_row) % rows_total;
    const uint8_t* g = src + r * pitch + (tid % per_row) * 16;
    uint32_t d = smem_u32(smem + ((i % (DEPTH + 1)) * blockDim.x + tid) * 16);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(g) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH) : "memory");
    row += stride;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (tid == 0) sink[blockIdx.x] = smem[7];
}

__global__ void __launch_bounds__(128, 1) probe_store(const __grid_constant__ CUtensorMap tm, int rows_total, int box_rows,
                                                       int box_bytes, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0) {
    int nblk = rows_total / box_rows;
    int b = blockIdx.x;
    for (int i = 0; i < iters; ++i) {
      bulk_wait_read<3>();
      tma_store_2d(&tm, smem + (i & 3) * box_bytes, 0, (b % nblk) * box_rows);
      bulk_commit();
      b += gridDim.x;
    }
    bulk_wait_all();
  }
}

int main(int argc, char** argv) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  const size_t bytes = (argc > 1 ? atoll(argv[1]) : 1024ll) << 20;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  cudaFuncSetAttribute(probe_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int inners[] = {16, 32, 64, 128, 256};
  const int rows_list[] = {32, 128, 256};
  for (int store = 0; store < 2; ++store)
    for (int inner : inners)
      for (int rows : rows_list) {
        const int row_bytes = inner * 2;
        const int box_bytes = row_bytes * rows;
        if (box_bytes * 4 > 190 * 1024) continue;
        // tensor: [rows_total][inner] with a row pitch of 512 B (like an NHWC activation)
        const int pitch = 512 > row_bytes ? 512 : row_bytes;
        const long long rows_total = (long long)(bytes / pitch) / rows * rows;
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows_total};
        cuuint64_t strides[1] = {(cuuint64_t)pitch};
        cuuint32_t box[2] = {(cuuint32_t)(inner > 256 ? 256 : inner), (cuuint32_t)rows};
        cuuint32_t es[2] = {1, 1};
        CUtensorMapSwizzle swz = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                   : CU_TENSOR_MAP_SWIZZLE_NONE;
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          printf("encode failed inner=%d rows=%d (%d)\n", inner, rows, (int)r);
          continue;
        }
        const int iters = (int)((256ll << 20) / box_bytes / 148) + 8;
        for (int S : {4, 8, 16}) {
          if (S * box_bytes > 190 * 1024 || (store && S != 4)) continue;
          float ms = 0;
          for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (store)
              probe_store<<<148, 128, 4 * box_bytes + 64>>>(tm, (int)rows_total, rows, box_bytes, iters);
            else
              probe_load<<<148, 128, S * box_bytes + 256>>>(tm, (int)rows_total, rows, box_bytes, iters, sink, S);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
          }
          cudaEventElapsedTime(&ms, e0, e1);
          const double moved = (double)iters * 148 * box_bytes;
          const double req = (double)iters * rows;  // rows per SM
          printf("%s S=%2d row %4d B x %3d rows: %7.1f GB/s total, %6.2f cycles/row/SM @1.9GHz\n",
                 store ? "STORE" : "LOAD ", S, row_bytes, rows, moved / ms / 1e6, ms * 1e-3 * 1.9e9 / req);
        }
      }
  cudaFuncSetAttribute(probe_cpasync<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe_cpasync<14>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe_cpasync<22>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int thr : {256, 512})
  for (int depth : {6, 14, 22})
  for (int rb : {128, 512}) {
    const int pitch = 512;
    const long long rows_total = (long long)(bytes / pitch);
    const int per_iter_bytes = thr * 16;
    const int iters = (int)((256ll << 20) / per_iter_bytes / 148);
    float ms = 0;
    const size_t sm = (size_t)(depth + 1) * thr * 16;
    if (sm > 200 * 1024) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (depth == 6) probe_cpasync<6><<<148, thr, sm>>>(reinterpret_cast<const uint8_t*>(buf), rows_total, pitch, rb, iters, sink);
      if (depth == 14) probe_cpasync<14><<<148, thr, sm>>>(reinterpret_cast<const uint8_t*>(buf), rows_total, pitch, rb, iters, sink);
      if (depth == 22) probe_cpasync<22><<<148, thr, sm>>>(reinterpret_cast<const uint8_t*>(buf), rows_total, pitch, rb, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("CPASYNC row %4d B, %d thr, %2d groups in flight (%6zu B/SM): %7.1f GB/s total\n", rb, thr, depth, (size_t)depth * thr * 16,
           (double)iters * 148 * per_iter_bytes / ms / 1e6);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
