// Shared device helpers for the sm_100a kernels: mbarriers, TMA, tcgen05/TMEM.
// Inline PTX only (no CUTLASS/CuTe dependency); encodings follow the PTX ISA
// tables for sm_100a (instruction descriptor for .kind::f16, shared-memory
// matrix descriptor version 1).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define UB_DEVI __device__ __forceinline__

namespace ub {

UB_DEVI uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// ---------------------------------------------------------------- mbarrier
UB_DEVI void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
UB_DEVI void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
UB_DEVI void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
UB_DEVI void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
UB_DEVI bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint (ns): the thread sleeps in hardware until the phase
// completes or the hint elapses -- for waiters that would otherwise spin for many
// microseconds and steal issue slots from the warps doing the work.
UB_DEVI bool mbar_try_wait_hint(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}
UB_DEVI void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait_hint(a, parity, ns)) return;
  long long t0 = clock64();
  while (!mbar_try_wait_hint(a, parity, ns)) {
    if (clock64() - t0 > (1ll << 33)) asm volatile("trap;");
  }
}

// Bounded wait: a lost arrival traps (kernel error) instead of hanging the GPU.
// UB_MBAR_HINT_NS > 0: the retry loop passes a suspend-time hint, so a waiting warp sleeps
// in hardware instead of re-polling (ncu: polling loops took a quarter of the issued
// instructions of a small-channel halo conv).
#ifndef UB_MBAR_HINT_NS
#define UB_MBAR_HINT_NS 0
#endif
UB_DEVI void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  long long t0 = clock64();
  while (!(UB_MBAR_HINT_NS ? mbar_try_wait_hint(a, parity, UB_MBAR_HINT_NS) : mbar_try_wait(a, parity))) {
    if (clock64() - t0 > (1ll << 33)) {  // ~4 s at 2 GHz
      asm volatile("trap;");
    }
  }
}

// ---------------------------------------------------------------- programmatic dependent launch
// Kernels of the forward are launched with programmatic stream serialisation (ub_host.h
// launch_pdl): a kernel may start -- barrier init, TMEM alloc, resident weights -- while
// its predecessor drains, and blocks in griddep_wait() before reading the predecessor's
// output.  Both are no-ops for a normal launch.
UB_DEVI void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
UB_DEVI void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- proxy fences
UB_DEVI void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------- TMA
UB_DEVI void tma_prefetch_desc(const void* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
UB_DEVI void tma_load_2d(const void* map, uint64_t* bar, void* smem, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
UB_DEVI void tma_load_3d(const void* map, uint64_t* bar, void* smem, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
UB_DEVI void tma_load_4d(const void* map, uint64_t* bar, void* smem, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
UB_DEVI void tma_load_im2col_4d(const void* map, uint64_t* bar, void* smem, int c, int w, int h, int n,
                                uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(off_w), "h"(off_h)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05 / TMEM
UB_DEVI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
UB_DEVI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Whole warp: allocate `ncols` (power of two >= 32) TMEM columns; address -> *slot.
UB_DEVI void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
UB_DEVI void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// Instruction descriptor, .kind::f16: bf16 x bf16 -> f32, both operands K-major.
//   [4,6) D fmt (1 = F32) | [7,10) A fmt (1 = BF16) | [10,13) B fmt (1 = BF16)
//   [15] A major (0 = K) | [16] B major (0 = K) | [17,23) N>>3 | [24,29) M>>4
UB_DEVI uint32_t make_idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// Shared-memory matrix descriptor (version 1), K-major, swizzled.
//   [0,14) start>>4 | [16,30) LBO>>4 (=1, unused for swizzled K-major)
//   [32,46) SBO>>4 (8 rows * row bytes) | [46,48) version = 1 | [61,64) layout
// layout: 2 = SWIZZLE_128B (64 bf16 per row), 6 = SWIZZLE_32B (16 bf16 per row).
UB_DEVI uint64_t make_sdesc(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(layout & 7u) << 61;
  return d;
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by ONE thread for the whole CTA.
UB_DEVI void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-wide forms: executed by all 32 (converged) lanes, ONE lane (elect.sync) issues.  Keeping
// the whole warp on the issue path lets the descriptors live in uniform registers; a
// lane-0-only branch makes the compiler wrap every MMA in a per-lane serialisation loop
// (measured on B200: 87 cycles per MMA issue from one lane vs 48 at N=64 / 64 at N=128 here).
UB_DEVI void umma_bf16_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
UB_DEVI void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// No-swizzle K-major shared-memory descriptor with explicit LBO (K-direction core-matrix
// stride) and SBO (8-row group stride): core matrices are 8 rows x 16 bytes.
UB_DEVI uint64_t sdesc_plain(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  return d;  // layout 0 = SWIZZLE_NONE
}

// 1-D bulk copy global -> shared, completion on an mbarrier (expect_tx by the caller).
UB_DEVI void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

UB_DEVI void tma_store_4d(const void* map, const void* smem, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

UB_DEVI void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Arrive on `bar` once all previously issued MMAs of this thread completed.
UB_DEVI void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Warp-collective: lanes (32*(warp%4) + i) of TMEM, 16 consecutive f32 columns.
UB_DEVI void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
// 16 columns into the first half of a 32-register array (keeps the array in registers)
UB_DEVI void tmem_ld16_lo(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
UB_DEVI void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- misc
UB_DEVI uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
UB_DEVI float2 unpack_bf16x2(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}

}  // namespace ub

namespace ub {
// ---------------------------------------------------------------- TMA store (bulk groups)
UB_DEVI void tma_store_2d(const void* map, const void* smem, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem)), "r"(c0), "r"(c1)
               : "memory");
}
UB_DEVI void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
UB_DEVI void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
UB_DEVI void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Warp-collective: 32 lanes x 32 consecutive f32 columns.
UB_DEVI void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
      " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
}  // namespace ub

namespace ub {
// ---------------------------------------------------------------- cp.async (LSU) producers
// 16-byte async copy global -> shared; src_bytes = 0 zero-fills the destination.
UB_DEVI void cp_async16(void* smem, const void* gmem, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
               : "memory");
}
UB_DEVI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
UB_DEVI void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Arrive on `bar` once all prior cp.async of this thread have landed (no pending-count increment).
UB_DEVI void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
}  // namespace ub

namespace ub {
// ---------------------------------------------------------------- packed math (sm_100: FADD2, HMNMX2)
UB_DEVI float2 add_f32x2(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
// bf16x2 (packed in a u32) -> float2, exact.
UB_DEVI float2 bf16x2_to_f32x2(uint32_t u) { return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u)); }
// max(x, 0) on a packed bf16x2; relu(round(x)) == round(relu(x)) so this is exact.
UB_DEVI uint32_t relu_bf16x2(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  v = __hmax2(v, __floats2bfloat162_rn(0.f, 0.f));
  return *reinterpret_cast<uint32_t*>(&v);
}
}  // namespace ub

namespace ub {
// Warp-collective: write 32 consecutive f32 columns of lanes (32*(warp%4) + i).
UB_DEVI void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0],"
      " {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16,"
      " %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
UB_DEVI void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// Round two f32 to a packed bf16x2 (lo, hi); with ReLU folded into the conversion.
UB_DEVI uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// Activation codes of include/upscale_b200.h (UB_ACT_*); conv epilogues take the code in
// their `relu` field (1 = ReLU keeps its packed cvt.relu fast path).
// tanh.approx.f32: one MUFU op (max relative error ~2^-11, far below the bf16 rounding that
// follows every activation here)
UB_DEVI float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
UB_DEVI float act_f(float v, int act) {
  switch (act) {
    case 1: return fmaxf(v, 0.f);
    case 2: return fminf(fmaxf(v, 0.f), 6.f);
    case 3: return v * fminf(fmaxf(v + 3.f, 0.f), 6.f) * (1.f / 6.f);
    case 4: return fminf(fmaxf(v + 3.f, 0.f), 6.f) * (1.f / 6.f);
    // SiLU / sigmoid through sigmoid(v) = (1 + tanh(v / 2)) / 2: one MUFU op per value instead
    // of exp + reciprocal (the SiLU conv epilogues were bound by the special-function unit)
    case 5: { const float h = 0.5f * v; return fmaf(h, tanh_fast(h), h); }
    case 6: return fmaf(0.5f, tanh_fast(0.5f * v), 0.5f);
    default: return v;
  }
}
// 8 fp32 -> activation -> 8 packed bf16, the activation switch resolved ONCE per call: a
// per-element switch on a runtime code (act_f) compiles to an indirect branch per value and
// serialises the epilogue's exp / reciprocal chains (ncu: a SiLU conv epilogue ran 4x slower
// than the ReLU one); here each case is straight-line code with 8 independent chains.
UB_DEVI uint64_t f2_bits(float lo, float hi) {
  return static_cast<uint64_t>(__float_as_uint(lo)) | (static_cast<uint64_t>(__float_as_uint(hi)) << 32);
}
// SiLU of a pair with the packed fp32x2 pipe (sm_100: mul / fma .f32x2 -- same rounding as the
// scalar ops, half the instructions): h = v/2, silu = h + h * tanh(h)
UB_DEVI uint32_t silu_bf16x2(float a, float b) {
  uint64_t h, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(h) : "l"(f2_bits(a, b)), "l"(f2_bits(0.5f, 0.5f)));
  const float hx = __uint_as_float(static_cast<uint32_t>(h)), hy = __uint_as_float(static_cast<uint32_t>(h >> 32));
  asm("fma.rn.f32x2 %0, %1, %2, %1;" : "=l"(r) : "l"(h), "l"(f2_bits(tanh_fast(hx), tanh_fast(hy))));
  return cvt_bf16x2(__uint_as_float(static_cast<uint32_t>(r)), __uint_as_float(static_cast<uint32_t>(r >> 32)));
}
template <int A>
UB_DEVI uint32_t act_pack2_c(float a, float b) {
  if (A == 5) return silu_bf16x2(a, b);
  return cvt_bf16x2(act_f(a, A), act_f(b, A));
}
UB_DEVI uint2 act_pack4(int act, float a, float b, float c, float d) {
  switch (act) {
    case 1: return make_uint2(act_pack2_c<1>(a, b), act_pack2_c<1>(c, d));
    case 2: return make_uint2(act_pack2_c<2>(a, b), act_pack2_c<2>(c, d));
    case 3: return make_uint2(act_pack2_c<3>(a, b), act_pack2_c<3>(c, d));
    case 4: return make_uint2(act_pack2_c<4>(a, b), act_pack2_c<4>(c, d));
    case 5: return make_uint2(act_pack2_c<5>(a, b), act_pack2_c<5>(c, d));
    case 6: return make_uint2(act_pack2_c<6>(a, b), act_pack2_c<6>(c, d));
    default: return make_uint2(act_pack2_c<0>(a, b), act_pack2_c<0>(c, d));
  }
}
// d = a * b + c on packed fp32 pairs (fma.rn.f32x2: the scalar fmaf rounding, one instruction)
UB_DEVI uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
UB_DEVI float f2_lo(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
UB_DEVI float f2_hi(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
template <int A>
UB_DEVI uint4 act_pack8_c(float f0, float f1, float f2, float f3, float f4, float f5, float f6, float f7) {
  return make_uint4(act_pack2_c<A>(f0, f1), act_pack2_c<A>(f2, f3), act_pack2_c<A>(f4, f5), act_pack2_c<A>(f6, f7));
}
UB_DEVI uint4 act_pack8(int act, float f0, float f1, float f2, float f3, float f4, float f5, float f6, float f7) {
  switch (act) {
    case 1: return act_pack8_c<1>(f0, f1, f2, f3, f4, f5, f6, f7);
    case 2: return act_pack8_c<2>(f0, f1, f2, f3, f4, f5, f6, f7);
    case 3: return act_pack8_c<3>(f0, f1, f2, f3, f4, f5, f6, f7);
    case 4: return act_pack8_c<4>(f0, f1, f2, f3, f4, f5, f6, f7);
    case 5: return act_pack8_c<5>(f0, f1, f2, f3, f4, f5, f6, f7);
    case 6: return act_pack8_c<6>(f0, f1, f2, f3, f4, f5, f6, f7);
    default: return act_pack8_c<0>(f0, f1, f2, f3, f4, f5, f6, f7);
  }
}
UB_DEVI uint32_t cvt_relu_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// Lane-wise max of three packed bf16x2 (exact).
UB_DEVI uint32_t bf16x2_max3(uint32_t a, uint32_t b, uint32_t c) {
  __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a);
  const __nv_bfloat162 y = *reinterpret_cast<__nv_bfloat162*>(&b);
  const __nv_bfloat162 z = *reinterpret_cast<__nv_bfloat162*>(&c);
  x = __hmax2(x, __hmax2(y, z));
  return *reinterpret_cast<uint32_t*>(&x);
}
}  // namespace ub
