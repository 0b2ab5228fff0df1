/* Profiling / self-test entry points of tools/libapmg_debug.so (built by `make`, never loaded by
 * the package): tcgen05 operand-layout self-tests and the roofline peak probes. */
#pragma once
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* tcgen05 kind::tf32 self-test (one CTA, one GEMM; umma_debug.cu) */
int apmg_debug_umma_gemm(int32_t cfg, int32_t K, int32_t N, int32_t split3, const float* A, const float* B,
                         float* D, void* stream);
/* 16-bit self-test (umma_bf16_debug.cu): D[M][N] = A[M][K] . B[K][N] (row-major f32 in),
 * bf16x3 operands, mode bit 0 = B MN-major, bit 1 = A MN-major, split3: 6 products */
int apmg_debug_umma_bf16(int32_t mode, int32_t M, int32_t K, int32_t N, int32_t split3, const float* A, const float* B,
                         float* D, void* stream);
/* roofline peak probes (peaks.cu, tools/peaks.py): kind 0 L2 float2 gather (7: float4), 1 L2 float2
 * RED (8: float4 RED), 2 FP32 FFMA, 3 FP64 DFMA, 4 tcgen05 kind::tf32, 5 warp shuffles, 6 smem
 * atomics; `table` is a device buffer of table_bytes (power of two) for the memory kinds (a sink
 * otherwise); *work receives the work unit count of the launch (bytes, REDs, FLOP, ...). */
int apmg_peak_probe(int32_t kind, void* table, int64_t table_bytes, int32_t iters, double* work, void* stream);
#ifdef __cplusplus
}
#endif
