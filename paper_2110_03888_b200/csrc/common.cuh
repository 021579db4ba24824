// Shared device helpers for the sm_100a kernels of the Pseudo-to-Real step.
// Everything here is raw PTX for Blackwell (tcgen05 / TMA / mbarrier); no
// CUTLASS types are used so the kernels stay self-contained.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define P2R_DEVICE __device__ __forceinline__

namespace p2r {

constexpr int kNumSMs = 148;  // B200; persistent grids that need co-residency use device_sms()

// SMs available to this context on the current device (MIG / green contexts can
// expose fewer than a full B200), cached per device.
inline int device_sms() {
  static int cache[16] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return kNumSMs;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
    cache[dev] = n;
  }
  return cache[dev];
}

P2R_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Explicit shared-space accesses (pointers derived from aligned uintptr_t math
// lose their address space and otherwise compile to generic LD/ST).
P2R_DEVICE void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
P2R_DEVICE float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
               : "memory");
  return v;
}
P2R_DEVICE void sts32f(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// ----------------------------------------------------------------------------
// Programmatic dependent launch. Kernels launched through p2r::launch_k (PDL
// attribute set) run their dependency-free setup, then pdl_wait() before the
// first global read of anything an earlier kernel in the stream may write.
// pdl_trigger() lets the next grid be scheduled once every CTA of this grid has
// issued it (its CTAs then take SMs as soon as ours exit).
// ----------------------------------------------------------------------------
P2R_DEVICE void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
P2R_DEVICE void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ----------------------------------------------------------------------------
// mbarrier
// ----------------------------------------------------------------------------
P2R_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
P2R_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
P2R_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
P2R_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
P2R_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ----------------------------------------------------------------------------
// TMA
// ----------------------------------------------------------------------------
P2R_DEVICE void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
P2R_DEVICE void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
P2R_DEVICE void tma_load_2d_warp(uint32_t smem_dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
      "}\n" ::"r"(smem_dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
P2R_DEVICE void mbar_arrive_expect_tx_warp(uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
      "}\n" ::"r"(bar),
      "r"(bytes)
      : "memory");
}
// TMA 2-D tile store shared -> global (bulk group of the issuing thread).
P2R_DEVICE void tma_store_2d(const CUtensorMap* map, uint32_t smem_src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_src), "r"(c0), "r"(c1)
               : "memory");
}
P2R_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N of this thread's bulk groups may still be reading shared memory
template <int N>
P2R_DEVICE void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
P2R_DEVICE void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (TMA)
P2R_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// 1-D bulk async copy global -> shared (16-byte aligned, bytes % 16 == 0),
// completion counted on `bar` (arrive.expect_tx by the issuing thread).
P2R_DEVICE void bulk_load(uint32_t smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ----------------------------------------------------------------------------
// tcgen05 (5th-gen tensor cores, accumulators in TMEM)
// ----------------------------------------------------------------------------
P2R_DEVICE void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
P2R_DEVICE void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
P2R_DEVICE void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
P2R_DEVICE void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate).
P2R_DEVICE void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05.mma have completed.
P2R_DEVICE void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Advance a SW128 smem descriptor by `bytes` (added to the >>4 start-address field).
P2R_DEVICE uint64_t desc_add(uint64_t d, uint32_t bytes) { return d + (bytes >> 4); }

// Warp-collective variants: all 32 lanes execute with warp-uniform operands
// (so they stay in uniform registers) and one elected lane issues. Called from
// lane-0-only code, a tcgen05.mma costs R2UR moves plus an elect loop per MMA,
// which bounds 128x64 MMAs at ~80 cycles of issue.
P2R_DEVICE void umma_bf16_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
P2R_DEVICE void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// ----------------------------------------------------------------------------
// CTA pair (cluster of 2, tcgen05 cta_group::2): the leader (rank 0) issues
// M=256 MMAs that read A/B halves from both CTAs' shared memory at the same
// offsets; every tcgen05 alloc/mma/commit of such a kernel uses cta_group::2.
// ----------------------------------------------------------------------------
P2R_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
P2R_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
P2R_DEVICE void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
P2R_DEVICE void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// Shared-window address of `bar` in the leader CTA of this pair (peer bit cleared).
P2R_DEVICE uint32_t pair_leader_addr(const void* bar) { return smem_u32(bar) & 0xFEFFFFFFu; }
// TMA 2-D load into this CTA's smem, completion bytes counted on the leader's barrier.
P2R_DEVICE void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
// Warp-collective TMA issue (one elected lane; operands warp-uniform).
P2R_DEVICE void tma_load_2d_pair_warp(uint32_t smem_dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n"
      "}\n" ::"r"(smem_dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
P2R_DEVICE void umma_bf16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once, when the leader's prior MMAs complete) on `bar` in both CTAs.
P2R_DEVICE void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .b16 m;\n"
      "mov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// Warp-collective pair variants (see umma_bf16_warp).
P2R_DEVICE void umma_bf16_pair_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                    uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
P2R_DEVICE void umma_commit_pair_warp(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .b16 m;\n"
      ".reg .pred e;\n"
      "mov.b16 m, 3;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// Arrive on the barrier at the same offset in CTA `rank` of the cluster.
// Relaxed: the only ordering needed is of prior tcgen05 ops (tcgen05.fence::
// before_thread_sync supplies it). A .release.cluster arrive compiles to
// MEMBAR.ALL.GPU and would hold the TMEM slot until the warp's global stores land.
P2R_DEVICE void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
P2R_DEVICE void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
P2R_DEVICE void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 32 registers per thread -> 32 lanes x 32 consecutive 32-bit columns.
P2R_DEVICE void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t* r) {
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
P2R_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05 "version 1"), SWIZZLE_128B.
//   K-major : rows of 128 B (64 bf16 along K), 8-row groups 1024 B apart (SBO).
//   MN-major: 64 MN-elements per 128 B row, rows = K; 8-row groups 1024 B apart
//             (SBO), MN atoms of 64 elements `lbo_bytes` apart (LBO).
P2R_DEVICE uint64_t make_sw128_desc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version = 1 (sm_100)
  d |= static_cast<uint64_t>(2) << 61;  // layout type = SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f16 with bf16 A/B and fp32 D.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                               // D format f32
         | (1u << 7)                             // A = bf16
         | (1u << 10)                            // B = bf16
         | ((a_mn ? 1u : 0u) << 15)              // A major
         | ((b_mn ? 1u : 0u) << 16)              // B major
         | ((static_cast<uint32_t>(N) >> 3) << 17)
         | ((static_cast<uint32_t>(M) >> 4) << 24);
}

// ----------------------------------------------------------------------------
// numerics shared by several kernels (exact-erf GELU, tensor.cpp:237-263)
// ----------------------------------------------------------------------------
// Exact (erf) GELU from one exp2: for z = |x|/sqrt(2), erfc(z)/2 = e t h(t) with
// e = exp(-x^2/2), t = 1/(1 + z/2) and h a degree-8 least-squares fit of
// erfcx(z)/(2t) on t in (0,1] (constants pre-folded). Phi(x) = 1 - erfc/2
// (x >= 0) or erfc/2; phi(x) = e / sqrt(2 pi) shares the exponential.
// |error| vs float64 erf: gelu < 4e-7, gelu' < 4e-7 (outputs are bf16-rounded);
// ~21 instructions, versus ~2x for the erff/expf pair.
// Phi(-|x|) = t * h(t) * e, t = 1/(1+|x|/(2 sqrt2)), e = exp(-x^2/2): one-ex2
// erfc fit (degree 8, |err| < 4e-7). The scalar and pair (sm_100 FP32x2:
// FFMA2/FMUL2, one issue slot for two lanes' worth of math -- the GELU
// epilogues are issue-bound) forms run the same operations in the same order
// with every fusion explicit (ptxas contracts f32x2 mul+add even with .rn), so
// all epilogue paths round identically. Returns th = t*h; e via reference.
P2R_DEVICE float gelu_th(float x, float& e) {
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(fabsf(x), 0.35355339059327373f, 1.0f)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"((x * x) * -0.72134752044448170f));
  float h = fmaf(-2.377655916e-02f, t, 1.178763658e-01f);
  h = fmaf(h, t, -2.006432861e-01f);
  h = fmaf(h, t, 9.842023998e-02f);
  h = fmaf(h, t, 8.996849880e-03f);
  h = fmaf(h, t, 9.415699542e-02f);
  h = fmaf(h, t, 1.228528991e-01f);
  h = fmaf(h, t, 1.410695761e-01f);
  h = fmaf(h, t, 1.410471797e-01f);
  return t * h;
}
P2R_DEVICE float2 gelu_th2(float2 x, float2& e) {
  float2 t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.x) : "f"(fmaf(fabsf(x.x), 0.35355339059327373f, 1.0f)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.y) : "f"(fmaf(fabsf(x.y), 0.35355339059327373f, 1.0f)));
  const float2 a = __fmul2_rn(__fmul2_rn(x, x), make_float2(-0.72134752044448170f, -0.72134752044448170f));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(a.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(a.y));
  auto c2 = [](float c) { return make_float2(c, c); };
  float2 h = __ffma2_rn(c2(-2.377655916e-02f), t, c2(1.178763658e-01f));
  h = __ffma2_rn(h, t, c2(-2.006432861e-01f));
  h = __ffma2_rn(h, t, c2(9.842023998e-02f));
  h = __ffma2_rn(h, t, c2(8.996849880e-03f));
  h = __ffma2_rn(h, t, c2(9.415699542e-02f));
  h = __ffma2_rn(h, t, c2(1.228528991e-01f));
  h = __ffma2_rn(h, t, c2(1.410695761e-01f));
  h = __ffma2_rn(h, t, c2(1.410471797e-01f));
  return __fmul2_rn(t, h);
}
// gelu(x) = x Phi(x) = relu(x) - |x| Phi(-|x|)
P2R_DEVICE float gelu_f(float v) {
  float e;
  const float he = gelu_th(v, e) * e;
  return fmaf(-fabsf(v), he, fmaxf(v, 0.0f));
}
P2R_DEVICE float2 gelu2(float2 x) {
  float2 e;
  const float2 he = __fmul2_rn(gelu_th2(x, e), e);
  return make_float2(fmaf(-fabsf(x.x), he.x, fmaxf(x.x, 0.0f)), fmaf(-fabsf(x.y), he.y, fmaxf(x.y, 0.0f)));
}
// gelu'(x) = Phi(x) + x phi(x);  Phi(x) = 0.5 + sign(x) (0.5 - th e)
P2R_DEVICE float gelu_grad_f(float v) {
  float e;
  const float th = gelu_th(v, e);
  const float m = __uint_as_float(__float_as_uint(fmaf(-th, e, 0.5f)) | (__float_as_uint(v) & 0x80000000u));
  return fmaf(v * e, 0.39894228040143268f, 0.5f + m);
}
// gelu and gelu' from ONE evaluation of the fit (the forward epilogue stores both:
// the backward then multiplies by the stored derivative); bitwise the values of
// gelu_f / gelu_grad_f (resp. gelu2 / gelu_grad2), which run the same operations
P2R_DEVICE float gelu_pair_f(float v, float& gd) {
  float e;
  const float th = gelu_th(v, e);
  const float he = th * e;
  const float m = __uint_as_float(__float_as_uint(fmaf(-th, e, 0.5f)) | (__float_as_uint(v) & 0x80000000u));
  gd = fmaf(v * e, 0.39894228040143268f, 0.5f + m);
  return fmaf(-fabsf(v), he, fmaxf(v, 0.0f));
}
P2R_DEVICE float2 gelu_grad2(float2 x);
P2R_DEVICE float2 gelu_pair2(float2 x, float2& gd) {
  float2 e;
  const float2 th = gelu_th2(x, e);
  const float2 he = __fmul2_rn(th, e);
  float2 m = __ffma2_rn(make_float2(-th.x, -th.y), e, make_float2(0.5f, 0.5f));
  m.x = __uint_as_float(__float_as_uint(m.x) | (__float_as_uint(x.x) & 0x80000000u));
  m.y = __uint_as_float(__float_as_uint(m.y) | (__float_as_uint(x.y) & 0x80000000u));
  const float2 cdf = __fadd2_rn(make_float2(0.5f, 0.5f), m);
  gd = __ffma2_rn(__fmul2_rn(x, e), make_float2(0.39894228040143268f, 0.39894228040143268f), cdf);
  return make_float2(fmaf(-fabsf(x.x), he.x, fmaxf(x.x, 0.0f)), fmaf(-fabsf(x.y), he.y, fmaxf(x.y, 0.0f)));
}
P2R_DEVICE float2 gelu_grad2(float2 x) {
  float2 e;
  const float2 th = gelu_th2(x, e);
  float2 m = __ffma2_rn(make_float2(-th.x, -th.y), e, make_float2(0.5f, 0.5f));  // >= 0
  m.x = __uint_as_float(__float_as_uint(m.x) | (__float_as_uint(x.x) & 0x80000000u));
  m.y = __uint_as_float(__float_as_uint(m.y) | (__float_as_uint(x.y) & 0x80000000u));
  const float2 cdf = __fadd2_rn(make_float2(0.5f, 0.5f), m);
  return __ffma2_rn(__fmul2_rn(x, e), make_float2(0.39894228040143268f, 0.39894228040143268f), cdf);
}

// 2^z on the FMA pipe (FP32x2), for softmax exponentials beyond what the SFU
// (16 ex2 / clk / SM on B200) sustains: z = n + f with n = round(z) via the
// 1.5*2^23 trick, 2^f by a degree-3 minimax polynomial (|rel err| < 1e-4: the
// results feed bf16 MMA operands), 2^n added to the exponent bits. z >= -125.
P2R_DEVICE float2 exp2_fma2(float2 z) {
  z.x = fmaxf(z.x, -125.0f);
  z.y = fmaxf(z.y, -125.0f);
  const float2 M = make_float2(12582912.0f, 12582912.0f);
  const float2 t = __fadd2_rn(z, M);
  const float2 nn = __ffma2_rn(t, make_float2(-1.0f, -1.0f), M);  // -n
  const float2 f = __fadd2_rn(z, nn);
  float2 q = __ffma2_rn(make_float2(5.502931029e-02f, 5.502931029e-02f), f,
                        make_float2(2.422568053e-01f, 2.422568053e-01f));
  q = __ffma2_rn(q, f, make_float2(6.932530403e-01f, 6.932530403e-01f));
  q = __ffma2_rn(q, f, make_float2(9.999513626e-01f, 9.999513626e-01f));
  constexpr uint32_t kMagicExp = 0x4B400000u << 23;  // (bits of M) << 23 mod 2^32: only the sum matters
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23) - kMagicExp),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23) - kMagicExp));
}
// Static boustrophedon schedule for persistent kernels over work items sorted
// heaviest-first: CTA c of G takes item c in round 0, G-1-c in round 1, ...
// (pairs heavy with light items; strictly increasing per CTA).
P2R_DEVICE int snake_item(int k, int c, int G) { return k * G + ((k & 1) ? G - 1 - c : c); }

P2R_DEVICE float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
P2R_DEVICE double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
P2R_DEVICE float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace p2r
