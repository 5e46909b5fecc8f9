// C-ABI plumbing: error reporting, launch counter, driver entry points.
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "ub_host.h"

namespace {
thread_local std::string g_err;
thread_local long long g_launches = 0;
std::once_flag g_once;
PFN_cuTensorMapEncodeTiled_v12000 g_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_im2col = nullptr;

void resolve() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
}
}  // namespace

namespace ub {

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return UB_OK;
  return fail(UB_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

void count_launch() { ++g_launches; }

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UB_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// Per-device state: one process may drive several GPUs (the C ABI does not assume one
// device per process), so SM counts and kernel attributes are kept per device ordinal.
namespace {
std::mutex g_dev_mu;
std::vector<int> g_sms;                                   // device -> SM count (0 = unknown)
std::vector<std::pair<int, const void*>> g_smem_done;     // (device, kernel) with max dyn smem set
}  // namespace

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

int num_sms() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (static_cast<int>(g_sms.size()) <= dev) g_sms.resize(dev + 1, 0);
  if (g_sms[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}

cudaError_t ensure_max_smem(const void* kernel, int bytes) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  for (const auto& e : g_smem_done)
    if (e.first == dev && e.second == kernel) return cudaSuccess;
  const cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err == cudaSuccess) g_smem_done.emplace_back(dev, kernel);
  return err;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled_fn() {
  std::call_once(g_once, resolve);
  return g_tiled;
}
PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col_fn() {
  std::call_once(g_once, resolve);
  return g_im2col;
}

}  // namespace ub

extern "C" {

const char* ub_last_error(void) { return g_err.c_str(); }
int ub_abi_version(void) { return 7; }
long long ub_launch_count(void) { return g_launches; }
void ub_reset_launch_count(void) { g_launches = 0; }

}  // extern "C"
