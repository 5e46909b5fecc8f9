// MUFU throughput probe (dev tool): tanh.approx / ex2.approx / rcp.approx per SM per clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_probe.cu -o mufu_probe && ./mufu_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void probe(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = 0.001f * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float y;
      if (OP == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(v[j]));
      if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[j]));
      if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[j]));
      if (OP == 3) asm volatile("fma.rn.f32 %0, %1, %1, %1;" : "=f"(y) : "f"(v[j]));
      v[j] = y * 0.5f;
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, float* d, int sms) {
  const int iters = 4096, blocks = sms * 4, threads = 512;
  probe<OP><<<blocks, threads>>>(d, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<OP><<<blocks, threads>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ops = (double)blocks * threads * iters * 8;
  printf("%-6s %8.1f Gop/s  %6.1f per SM per clock (at %d MHz)\n", name, ops / ms / 1e6,
         ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, sms * 4 * 512 * sizeof(float));
  run<0>("tanh", d, sms);
  run<1>("ex2", d, sms);
  run<2>("rcp", d, sms);
  run<3>("ffma", d, sms);
  return 0;
}
