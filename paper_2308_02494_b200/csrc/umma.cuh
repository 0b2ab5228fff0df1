// tcgen05 (5th-gen tensor core) building blocks for sm_100a, written against the
// PTX ISA directly: shared-memory matrix descriptors, instruction descriptors,
// kind::tf32 MMA issue, commit-to-mbarrier, TMEM allocation and loads.
//
// Operand layout ("CM layout"): a row-major matrix X[R][C] of 32-bit values is
// stored as 8x16-byte core matrices,
//     offset(r, c) = (c/4)*SC + (r/8)*128 + (r%8)*16 + (c%4)*4,   SC = R*16,
// the canonical K-major SWIZZLE_NONE layout with rows = M/N and cols = K (SBO = 128 B
// between 8-row groups, LBO = SC between the two 16-B K chunks of one K=8 tf32 MMA);
// a thread owning a row writes whole 16-byte chunks (conflict-free).
//
// kind::tf32 reads MN-major operands only in the 128B-with-32B-atom swizzle (CUTLASS:
// "SW128_32B is the only available smem layout" for MN-major tf32), whose physical
// arrangement differs from every K-major one, so a matrix needed in both orientations
// takes two copies.  The fused recon kernel instead keeps the transposed weights in
// tensor memory and issues those products with the A operand from TMEM (mma_tf32_ts).
#pragma once

#include <stdint.h>
#include <cuda_bf16.h>

namespace apmg {
namespace umma {

__host__ __device__ constexpr uint32_t cm_offset(int r, int c, int R) {
  return uint32_t((c >> 2) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (c & 3) * 4);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SWIZZLE_NONE shared-memory descriptor (Blackwell version 1).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version = 1 (sm_100)
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0 (SWIZZLE_NONE)
  return d;
}

// Descriptor of a CM-layout buffer used K-major (rows = M or N) at K-step kk (K=8 each).
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int R, int kk) {
  return smem_desc(base + uint32_t(kk) * 2u * uint32_t(R * 16), uint32_t(R * 16), 128u);
}
// SWIZZLE_NONE MN-major descriptor of a CM-layout buffer (cols = M or N, rows = K) at K-step
// kk.  Kept for the self-test only: kind::tf32 does not accept this layout (see above).
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int R, int kk) {
  return smem_desc(base + uint32_t(kk) * 128u, 128u, uint32_t(R * 16));
}

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                      // c_format = F32
         | (2u << 7)                    // a_format = TF32
         | (2u << 10)                   // b_format = TF32
         | (uint32_t(a_mn) << 15)       // a_major (0 = K, 1 = MN)
         | (uint32_t(b_mn) << 16)       // b_major
         | (uint32_t(N >> 3) << 17)     // n_dim
         | (uint32_t(M >> 4) << 24);    // m_dim
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// same, with the explicit (all-enabled) disable-output-lane mask operand
__device__ __forceinline__ void mma_tf32_mask(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(z));
}

// A operand from tensor memory (M=128: row m in lane m, K elements in consecutive columns).
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// ---- 16-bit operands (kind::f16 with BF16 inputs, F32 accumulate) ----
// CM layout for 2-byte elements: 8 rows x 16 B (8 elements) core matrices,
//     byte offset(r, c) = (c/8)*R*16 + (r/8)*128 + (r%8)*16 + (c%8)*2,
// K-major with rows = M/N (desc_kmajor: one K=16 MMA spans two 16-B chunks, like K=8 tf32)
// and, for 16-bit types, also usable MN-major with rows = K (desc_mnmajor16).
__host__ __device__ constexpr uint32_t cm16_offset(int r, int c, int R) {
  return uint32_t((c >> 3) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}
// MN-major descriptor at K-step kk (K=16 = two 8-row groups, 128 B apart)
__device__ __forceinline__ uint64_t desc_mnmajor16(uint32_t base, int R, int kk) {
  return smem_desc(base + uint32_t(kk) * 256u, 128u, uint32_t(R * 16));
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                      // c_format = F32
         | (1u << 7)                    // a_format = BF16
         | (1u << 10)                   // b_format = BF16
         | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Descriptors as (runtime base) + (compile-time fields): DescC holds the low word without
// the base, (offset >> 4) | (LBO >> 4) << 16, and the high word (SBO >> 4) | version.  The
// issuing thread adds base16 = (smem window address >> 4) per operand -- one integer add per
// MMA operand instead of re-deriving and masking every field (the single issuing thread is
// on the critical path of the small M=64 products).  Valid while offsets stay < 256 KB.
struct DescC {
  uint32_t lo, hi;
};
__host__ __device__ constexpr DescC kmajor_c(uint32_t off, int R, int kk) {
  return DescC{((off + uint32_t(kk) * 2u * uint32_t(R * 16)) >> 4) | ((uint32_t(R * 16) >> 4) << 16),
               (128u >> 4) | (1u << 14)};
}
__host__ __device__ constexpr DescC mnmajor16_c(uint32_t off, int R, int kk) {
  return DescC{((off + uint32_t(kk) * 256u) >> 4) | ((128u >> 4) << 16), (uint32_t(R * 16) >> 4) | (1u << 14)};
}
__device__ __forceinline__ void mma_bf16_c(uint32_t d_tmem, uint32_t base16, DescC a, DescC b, uint32_t idesc,
                                           uint32_t accumulate) {
#ifdef APMG_ABL_NOMMA  // timing ablation only: no tensor-core work (wrong results)
  if (idesc != 0xffffffffu) return;
#endif
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "mov.b64 da, {%1, %2};\n\t"
      "mov.b64 db, {%3, %4};\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}\n" ::"r"(d_tmem),
      "r"(base16 + a.lo), "r"(a.hi), "r"(base16 + b.lo), "r"(b.hi), "r"(idesc), "r"(accumulate));
}

// x = h + m + l in bf16 (8+8+8 significant bits: the f32 significand, exponent permitting)
__device__ __forceinline__ void split_bf16x3(float x, __nv_bfloat16& h, __nv_bfloat16& m, __nv_bfloat16& l) {
  h = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(h);
  m = __float2bfloat16_rn(r1);
  l = __float2bfloat16_rn(r1 - __bfloat162float(m));
}

// bf16x3 split of a pair (packed cvt.rn.bf16x2.f32 and fp32x2 residuals), as 3 packed words
__device__ __forceinline__ void split2_bf16x3(float x0, float x1, uint32_t& h, uint32_t& m, uint32_t& l) {
  const __nv_bfloat162 bh = __float22bfloat162_rn(make_float2(x0, x1));
  const float2 r1 = __fadd2_rn(make_float2(x0, x1), make_float2(-__low2float(bh), -__high2float(bh)));
  const __nv_bfloat162 bm = __float22bfloat162_rn(r1);
  const float2 r2 = __fadd2_rn(r1, make_float2(-__low2float(bm), -__high2float(bm)));
  const __nv_bfloat162 bl = __float22bfloat162_rn(r2);
  h = *reinterpret_cast<const uint32_t*>(&bh);
  m = *reinterpret_cast<const uint32_t*>(&bm);
  l = *reinterpret_cast<const uint32_t*>(&bl);
}

// write 8 consecutive columns (one 16-B chunk per plane) of row r of a bf16x3 CM buffer
__device__ __forceinline__ void store_chunk3(unsigned char* buf, uint32_t plane, int r, int c0, int R, const float* v) {
  uint32_t h[4], m[4], l[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) split2_bf16x3(v[2 * e], v[2 * e + 1], h[e], m[e], l[e]);
  const uint32_t o = umma::cm16_offset(r, c0, R);
  *reinterpret_cast<uint4*>(buf + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(buf + plane + o) = make_uint4(m[0], m[1], m[2], m[3]);
  *reinterpret_cast<uint4*>(buf + 2 * plane + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

// two adjacent columns (c even) of row r of a bf16x3 CM buffer: one 4-byte word per plane
__device__ __forceinline__ void store_pair3(unsigned char* buf, uint32_t plane, int r, int c, int R, float x0,
                                           float x1) {
  uint32_t h, m, l;
  split2_bf16x3(x0, x1, h, m, l);
  const uint32_t o = cm16_offset(r, c, R);
  *reinterpret_cast<uint32_t*>(buf + o) = h;
  *reinterpret_cast<uint32_t*>(buf + plane + o) = m;
  *reinterpret_cast<uint32_t*>(buf + 2 * plane + o) = l;
}

// same, high and middle planes only (operands of the 3-product backward)
__device__ __forceinline__ void store_pair2(unsigned char* buf, uint32_t plane, int r, int c, int R, float x0,
                                           float x1) {
  uint32_t h, m, l;
  split2_bf16x3(x0, x1, h, m, l);
  const uint32_t o = cm16_offset(r, c, R);
  *reinterpret_cast<uint32_t*>(buf + o) = h;
  *reinterpret_cast<uint32_t*>(buf + plane + o) = m;
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Every CTA warp waits here while the tensor core runs; probes take issue slots and shared-memory
// wavefronts from the warps that still have CUDA-core work. Default: probe, then sleep 32 ns between
// probes. A/B: APMG_MBAR_SLEEP=0 -> try_wait with a suspend-time hint (10 ms; in practice it returns
// after a short time, ~20 probes per wait), APMG_MBAR_SPIN=1 -> plain spin.
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  const uint32_t a = smem_u32(mbar);
#ifndef APMG_MBAR_SLEEP
#define APMG_MBAR_SLEEP 32
#endif
#if APMG_MBAR_SLEEP > 0  // poll, back off APMG_MBAR_SLEEP ns between probes (-DAPMG_MBAR_SLEEP=0: the
                         // suspend-hint wait below): +0.6% on the recon kernel, whose 16 worker warps'
                         // probes were ~6% of its instructions and its shared-memory wavefronts
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(APMG_MBAR_SLEEP);
  }
#elif defined(APMG_MBAR_SPIN) && APMG_MBAR_SPIN
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 10000000;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(parity)
      : "memory");
#endif
}

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}
// named barrier over `count` threads (a subset of the CTA, e.g. the worker warps)
// signal a named barrier without waiting for it (the waiting side uses named_sync)
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// whole warp: allocate `cols` TMEM columns, address written to *dst (smem)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread (thread t <-> lane base + t)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 lanes x 256 bit shape (M=64 accumulators: all 32 threads carry data).  Thread t gets
// rows t/4 and t/4 + 8 of the 16-lane block, columns 2(t%4) and 2(t%4)+1 of each 8-column
// repetition: v[4r+0] = (t/4, 8r+2(t%4)), v[4r+1] = (t/4, +1), v[4r+2] = (t/4+8, ..), v[4r+3]
// (the mma.sync accumulator fragment layout; probed on B200).
__device__ __forceinline__ void tmem_ld_16x256b_x2(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3]));
}
// 12 consecutive columns (x8 + x4), completion waited
__device__ __forceinline__ void tmem_ld12u(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
               : "r"(taddr + 8));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16u(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// round-to-nearest TF32 (the value the tensor core multiplies exactly) and the exact residual
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = tf32_rn(x);
  lo = x - hi;
}

// TMEM address of (lane, column) relative to the allocation base
__device__ __forceinline__ uint32_t taddr(uint32_t base, uint32_t lane, uint32_t col) {
  return base + (lane << 16) + col;
}

}  // namespace umma
}  // namespace apmg
