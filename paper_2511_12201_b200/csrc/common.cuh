// Shared device helpers for libomnisparse (sm_100a only).
//
// Thin inline-PTX wrappers for the Blackwell primitives the kernels use:
// mbarrier pipelines, TMA tile loads (cp.async.bulk.tensor), tcgen05 MMA with
// TMEM accumulators, TMEM load/store, and the proxy/ordering fences between
// them. Encodings follow the PTX ISA (tcgen05 shared-memory and instruction
// descriptors); bit layouts were cross-checked against the CUTLASS headers
// vendored with flashinfer (cute/arch/mma_sm100_desc.hpp).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <type_traits>

#include "../../include/omnisparse.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libomnisparse targets sm_100a only"
#endif

#define OMNI_CUDA_TRY(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) {                                  \
      omni_set_cuda_error(#expr, _e);                         \
      return OMNI_E_CUDA;                                     \
    }                                                         \
  } while (0)

#define OMNI_CHECK(cond, code, msg)                           \
  do {                                                        \
    if (!(cond)) {                                            \
      omni_set_last_error(msg);                               \
      return (code);                                          \
    }                                                         \
  } while (0)

// Defined in capi.cu: thread-local last-error string for diagnostics.
void omni_set_last_error(const char* msg);
void omni_set_cuda_error(const char* what, cudaError_t e);  // "<what>: <CUDA error string>"

// Every C-ABI entry point starts here: clears a non-sticky error another
// runtime call of this thread left behind (torch, CUB dispatch), so the
// launch check after our own launches reports only our launches.
static inline void omni_begin() { (void)cudaGetLastError(); }

// Defined in capi.cu: raises the dynamic shared-memory limit of kernel `fn`
// to at least `bytes` on the CURRENT device (the limit only grows); the
// attribute is per device context, so a process driving two GPUs sets it on
// each. Thread-safe.
cudaError_t omni_smem_attr_raw(const void* fn, int bytes);
template <typename F>
static inline cudaError_t omni_smem_attr(F* fn, int bytes) {
  return omni_smem_attr_raw(reinterpret_cast<const void*>(fn), bytes);
}

static inline int omni_launch_check() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    omni_set_cuda_error("kernel launch", e);
    return OMNI_E_CUDA;
  }
  return OMNI_OK;
}

namespace omni {

constexpr double kLog2e = 1.4426950408889634;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <typename T>
__device__ __forceinline__ double to_f64(T x);
template <>
__device__ __forceinline__ double to_f64<float>(float x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ double to_f64<double>(double x) { return x; }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 x) {
  return static_cast<double>(__bfloat162float(x));
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
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
// Blocking wait on the completion of the phase with parity `parity`. A
// watchdog turns a protocol deadlock into a trapped kernel (a CUDA error the
// host reports) instead of a hung device.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > (1LL << 33)) {
      printf("omnisparse: mbarrier watchdog fired (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}

// ----------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

// -------------------------------------------------------------------- fences
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---------------------------------------------------------------------- TMEM
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets lane
// (warp%4)*32 + t, columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void reg_fence16(uint32_t* r) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Register fence for software-pipelined TMEM loads: after tcgen05.wait::ld,
// route the destination registers of an in-flight tcgen05.ld through an empty
// volatile asm so no consumer is scheduled above the wait.
__device__ __forceinline__ void reg_fence32(uint32_t* r) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// --------------------------------------------------------------- tcgen05.mma
// Shared-memory matrix descriptor (sm_100 "version 1"): start address,
// leading/stride byte offsets (16-byte units), SWIZZLE_128B layout type (2).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version for tcgen05
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f16: bf16 A/B, fp32 accumulator, MxN tile.
// a_mn / b_mn select MN-major (transposed) operands.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)                                  // D format: f32
         | (1u << 7)                                // A format: bf16
         | (1u << 10)                               // B format: bf16
         | (static_cast<uint32_t>(a_mn) << 15)      // A major
         | (static_cast<uint32_t>(b_mn) << 16)      // B major
         | (static_cast<uint32_t>(N >> 3) << 17)    // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);   // M / 16
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Same with the A operand read from TMEM (K-major bf16 pairs, lane = row).
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once) on an mbarrier when all previously issued tcgen05 ops of this
// thread complete.
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Warp-converged variants: the whole warp executes the call (so descriptor
// arithmetic stays warp-uniform and lives in uniform registers) and
// elect.sync picks the one lane that issues the tcgen05 instruction.
__device__ __forceinline__ void umma_bf16_ws(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_ts_ws(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_ws(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}

// ------------------------------------------------- CTA pair (cta_group::2)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared-memory offset in CTA `rank`.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t ld_shared_cluster_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
// Arrive on an mbarrier in another CTA of the cluster (release, cluster scope).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Relaxed remote arrive: for signalling data whose writes are already
// complete (tcgen05.wait::st), without the cost of a cluster-scope release.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Wait with cluster-scope acquire (arrivals come from the peer CTA too).
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  if (mbar_try_wait_cluster(bar, parity)) return;
  long long t0 = clock64();
  while (!mbar_try_wait_cluster(bar, parity)) {
    if (clock64() - t0 > (1LL << 33)) {
      printf("omnisparse: cluster mbarrier watchdog fired (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}
// 2-SM TMA tile load: lands in this CTA's shared memory, completes the
// transaction bytes on the pair leader's mbarrier (peer bit of the address
// cleared, as CUTLASS's SM100_TMA_2SM_LOAD does).
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(dst),
      "l"(map), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish_pair() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// Pair MMA with A from TMEM (M = 256 across the two CTAs' lanes), B from each
// CTA's shared memory (N split between the CTAs), issued by the leader's
// elected lane; the whole warp calls it.
__device__ __forceinline__ void umma_pair_ts_ws(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Pair MMA with both operands in shared memory: A = this CTA's 128 rows in
// each CTA (same offset), B split along N between the CTAs.
__device__ __forceinline__ void umma_pair_ss_ws(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Commit of the leader's pair MMAs, arriving on the mbarrier at the same
// offset in both CTAs of the pair.
__device__ __forceinline__ void umma_commit_pair_ws(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 rx;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(bar)
      : "memory");
}

// --------------------------------------------------------------- misc math
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// 2^d for integral d <= 0 (exact; 0 below the normal range, and for -inf).
__device__ __forceinline__ float pow2_int(float d) {
  return d < -126.f ? 0.f : __int_as_float((static_cast<int>(d) + 127) << 23);
}
__device__ __forceinline__ uint32_t mul_bf16x2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// 2^x on the FMA/ALU pipes (no MUFU): round-to-nearest split x = n + f,
// f in [-0.5, 0.5], degree-3 relative-minimax polynomial (max rel err 7.5e-5,
// below the bf16 rounding P receives). Valid for x <= 127; -inf -> 0.
__device__ __forceinline__ float exp2_poly(float x) {
  const bool zero = x < -126.f;  // masked (-inf) and underflowing entries are exactly 0
  x = fmaxf(x, -126.f);
  const float r = x + 12582912.f;  // 1.5 * 2^23: integer part lands in the low mantissa bits
  const float f = x - (r - 12582912.f);
  float p = fmaf(0.05517165f, f, 0.24261116f);
  p = fmaf(p, f, 0.69326099f);
  p = fmaf(p, f, 0.99992807f);
  const float v = __int_as_float(__float_as_int(p) + ((__float_as_int(r) - 0x4B400000) << 23));
  return zero ? 0.f : v;
}

// ---- packed fp32 pairs (sm_100 FFMA2 / FADD2): lo = first element
__device__ __forceinline__ uint64_t f32x2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f32x2_lo(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return lo;
}
__device__ __forceinline__ float f32x2_hi(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return hi;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void mbar_inval(uint32_t bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// exp2 of a pair on the FMA pipe (same polynomial as exp2_poly); arguments
// below -126 (masked -inf included) give exactly 0.
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
  const float xl = f32x2_lo(x), xh = f32x2_hi(x);
  float lo = fmaxf(xl, -126.f), hi = fmaxf(xh, -126.f);
  const uint64_t xc = f32x2(lo, hi);
  const uint64_t magic = f32x2(12582912.f, 12582912.f), nmagic = f32x2(-12582912.f, -12582912.f);
  const uint64_t r = fadd2(xc, magic);            // integer part in the low mantissa bits
  const uint64_t f = fadd2(xc, fadd2(r, nmagic) ^ 0x8000000080000000ull);  // x - (r - magic), in [-0.5, 0.5]
  uint64_t p = ffma2(f32x2(0.05517165f, 0.05517165f), f, f32x2(0.24261116f, 0.24261116f));
  p = ffma2(p, f, f32x2(0.69326099f, 0.69326099f));
  p = ffma2(p, f, f32x2(0.99992807f, 0.99992807f));
  // scale by 2^n: (bits(r) - bits(magic)) << 23 == bits(r) << 23 (mod 2^32)
  const uint32_t rl = static_cast<uint32_t>(r), rh = static_cast<uint32_t>(r >> 32);
  const uint32_t pl = static_cast<uint32_t>(p), ph = static_cast<uint32_t>(p >> 32);
  const uint32_t ol = xl < -126.f ? 0u : pl + (rl << 23), oh = xh < -126.f ? 0u : ph + (rh << 23);
  return (static_cast<uint64_t>(oh) << 32) | static_cast<uint64_t>(ol);
}

// exp2 of a pair on the FMA/ALU pipes in 10 issue slots: clamp at -126,
// round-to-nearest split x = n + f with the 1.5 * 2^23 magic constant,
// degree-3 minimax polynomial for 2^f (max rel err 7.5e-5, far below the
// bf16 rounding P receives), n added straight into the exponent field
// ((bits(x + magic) << 23) == n << 23 mod 2^32). The caller guarantees no
// masked (-inf) entries: for x < -126 the result is 2^-126-ish, not 0.
struct Exp2PolyConsts {
  uint64_t magic, c3, c2, c1, c0;
};
__host__ __device__ inline Exp2PolyConsts exp2_poly_consts() {
  auto pr = [](float v) {
    uint32_t b;
    memcpy(&b, &v, 4);
    return (static_cast<uint64_t>(b) << 32) | b;
  };
  return {pr(12582912.f), pr(0.05517165f), pr(0.24261116f), pr(0.69326099f), pr(0.99992807f)};
}
__device__ __forceinline__ uint64_t exp2_poly_pair(uint64_t x, const Exp2PolyConsts& k) {
  uint64_t y;
  asm("{\n\t"
      ".reg .f32 xl, xh;\n\t"
      ".reg .b64 xc, r, t, f, p;\n\t"
      ".reg .b32 rl, rh, pl, ph;\n\t"
      "mov.b64 {xl, xh}, %1;\n\t"
      "max.f32 xl, xl, 0fC2FC0000;\n\t"
      "max.f32 xh, xh, 0fC2FC0000;\n\t"
      "mov.b64 xc, {xl, xh};\n\t"
      "add.rn.f32x2 r, xc, %2;\n\t"
      "sub.rn.f32x2 t, r, %2;\n\t"
      "sub.rn.f32x2 f, xc, t;\n\t"
      "fma.rn.f32x2 p, f, %3, %4;\n\t"
      "fma.rn.f32x2 p, p, f, %5;\n\t"
      "fma.rn.f32x2 p, p, f, %6;\n\t"
      "mov.b64 {rl, rh}, r;\n\t"
      "mov.b64 {pl, ph}, p;\n\t"
      "mad.lo.u32 pl, rl, 8388608, pl;\n\t"
      "mad.lo.u32 ph, rh, 8388608, ph;\n\t"
      "mov.b64 %0, {pl, ph};\n\t"
      "}"
      : "=l"(y)
      : "l"(x), "l"(k.magic), "l"(k.c3), "l"(k.c2), "l"(k.c1), "l"(k.c0));
  return y;
}

// Degree-2 variant (max rel err 1.7e-3, about bf16's half ulp): one FMA
// fewer per pair. Same clamp, split and exponent insertion as exp2_poly_pair.
__device__ __forceinline__ uint64_t exp2_poly2_pair(uint64_t x, const Exp2PolyConsts& k) {
  uint64_t y;
  asm("{\n\t"
      ".reg .f32 xl, xh;\n\t"
      ".reg .b64 xc, r, t, f, p;\n\t"
      ".reg .b32 rl, rh, pl, ph;\n\t"
      "mov.b64 {xl, xh}, %1;\n\t"
      "max.f32 xl, xl, 0fC2FC0000;\n\t"
      "max.f32 xh, xh, 0fC2FC0000;\n\t"
      "mov.b64 xc, {xl, xh};\n\t"
      "add.rn.f32x2 r, xc, %2;\n\t"
      "sub.rn.f32x2 t, r, %2;\n\t"
      "sub.rn.f32x2 f, xc, t;\n\t"
      "fma.rn.f32x2 p, f, %3, %4;\n\t"
      "fma.rn.f32x2 p, p, f, %5;\n\t"
      "mov.b64 {rl, rh}, r;\n\t"
      "mov.b64 {pl, ph}, p;\n\t"
      "mad.lo.u32 pl, rl, 8388608, pl;\n\t"
      "mad.lo.u32 ph, rh, 8388608, ph;\n\t"
      "mov.b64 %0, {pl, ph};\n\t"
      "}"
      : "=l"(y)
      : "l"(x), "l"(k.magic), "l"(0x3E7426333E742633ull), "l"(0x3F3414FE3F3414FEull), "l"(0x3F800E853F800E85ull));
  return y;
}


// Vector fp32 reduction into global memory (no return value).
__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// Named barrier with an OR reduction of a per-thread predicate.
__device__ __forceinline__ bool named_bar_red_or(uint32_t id, uint32_t nthreads, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 q, %3, 0;\n\t"
      "barrier.cta.red.or.pred p, %1, %2, q;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(id), "r"(nthreads), "r"(pred ? 1u : 0u)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Number of entries of ascending `a[0..n)` that are <= key (upper bound).
__device__ __forceinline__ int count_le(const int32_t* __restrict__ a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(a + mid) <= key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// count_le for the 32 ascending keys of a warp (invalid lanes: any key,
// result unused), warp-cooperatively: a 32-ary search for the first element
// >= the smallest key (one round of 32 parallel loads per level instead of 5
// dependent binary-search steps), then a scan of the window up to the
// largest key, 32 elements per load.
__device__ __forceinline__ int count_le_warp(const int32_t* __restrict__ a, int n, int key, bool valid) {
  const int lane = threadIdx.x & 31;
  int kmin = valid ? key : INT_MAX, kmax = valid ? key : INT_MIN;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (kmin == INT_MAX) return 0;
  int lo = 0, hi = n;  // the first index with a[k] >= kmin lies in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int idx = lo + lane * step;
    const int v = idx < hi ? __ldg(a + idx) : INT_MAX;
    const int k = __popc(__ballot_sync(0xffffffffu, v < kmin));  // pivots below kmin (a prefix)
    const int nlo = k == 0 ? lo : lo + (k - 1) * step + 1;
    hi = min(hi, lo + k * step);
    lo = nlo;
  }
  {
    const int idx = lo + lane;
    const int v = idx < hi ? __ldg(a + idx) : INT_MAX;
    lo += __popc(__ballot_sync(0xffffffffu, v < kmin));
  }
  int c = lo;  // every element below lo is < kmin <= key
  for (int base = lo; base < n; base += 32) {
    const int idx = base + lane;
    const int v = idx < n ? __ldg(a + idx) : INT_MAX;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const int kq = __shfl_sync(0xffffffffu, key, q);
      const int cnt = __popc(__ballot_sync(0xffffffffu, v <= kq));
      if (lane == q) c += cnt;
    }
    if (__shfl_sync(0xffffffffu, v, 31) > kmax) break;  // the window is exhausted
  }
  return c;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace omni
