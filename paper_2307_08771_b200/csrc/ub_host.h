// Host-side plumbing shared by the C-ABI translation units: thread-local error
// state, launch counting, and TMA descriptor encoding through the driver entry
// points (resolved at run time, so the .so does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <utility>

#include "upscale_b200.h"

namespace ub {

int fail(int code, const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);  // UB_OK or UB_ECUDA with message
void count_launch();

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled_fn();
PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col_fn();
// Clear the descriptor bit CUTLASS clears for small tensors on drivers <= 13.1.
void apply_small_tensor_quirk(CUtensorMap* map, size_t footprint_bytes);
int num_sms();  // multiprocessors of the current device (cached per device)
int current_device();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel).
cudaError_t ensure_max_smem(const void* kernel, int bytes);
template <typename... A>
cudaError_t ensure_max_smem(void (*kernel)(A...), int bytes = 227 * 1024) {
  return ensure_max_smem(reinterpret_cast<const void*>(kernel), bytes);
}
// Stride-1 3x3 halo-tile kernel (conv_halo.cu); *handled = false when the layer is outside
// its scope and the generic kernel should run instead.
int conv_halo_fwd(const ub_conv_desc* d, int lead, int cpad, cudaStream_t stream, bool* handled);

// Swizzle span in bytes -> CUtensorMapSwizzle.
inline CUtensorMapSwizzle swizzle_of(int bytes) {
  switch (bytes) {
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    default: return CU_TENSOR_MAP_SWIZZLE_NONE;
  }
}

// Grid for a grid-stride loop over `work` items: at most 16 CTAs per SM.
inline int grid_for(long long work, int block, int per_thread = 1) {
  long long g = (work + (long long)block * per_thread - 1) / ((long long)block * per_thread);
  const long long cap = (long long)num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// Launch with programmatic stream serialisation (PDL) unless UB_PDL=0: the kernel may begin
// while the previous kernel on the stream finishes; it must call griddep_wait() before
// consuming that kernel's results.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// L2 promotion for activation tensor maps (conv_tc.cu): 256 B for rows read whole, else 64 B.
CUtensorMapL2promotion a_promo(bool whole_rows);

}  // namespace ub
