/*
 * slora_oracle.h -- CPU fp64 ORACLE for S-LoRA's heterogeneous batched LoRA
 * (arXiv 2311.03285).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path under
 * paper_2311_03285_b200/ and include/; neither side includes the other.
 *
 * Citations: P:L = /root/reference/PAPER.md line L (read-only at build time,
 * absent on the GPU box; citations are documentation only).
 *
 * What is computed (the plain definition; the method reaches exactly this up
 * to rounding order):
 *   Eq. (lora_factored), P:121   h = xW + xAB,  W in R^{h x d}, A in R^{h x r},
 *                                B in R^{r x d}
 *   per token i with adapter a = slot[i] ("compute xAB on the fly")
 *     v_i[j]   = sum_{k=0}^{h-1} x[i,k] * A_a[k,j]       (k ascending)
 *     delta[c] = sum_{j=0}^{r_a-1} v_i[j] * B_a[j,c]      (j ascending)
 *     out_i    = y_in_i + scale_a * delta                  (scale: DESIGN.md R6)
 *   a token with slot -1 has no adapter: out_i = y_in_i     (R7)
 *
 * All arrays are dense, row-major fp64, UNPAGED (the oracle never sees the
 * unified pool).  A_all/B_all hold every adapter's A (h x r_a) and B (r_a x d)
 * back to back at element offsets A_off[a], B_off[a].
 *
 * Threads: tokens are split into disjoint contiguous ranges, one pthread
 * each; a token's arithmetic is identical for every thread count.
 * Return value: 0 on success, -1 on a bad argument (negative size, slot out
 * of range, rank < 1).
 */
#ifndef SLORA_ORACLE_H
#define SLORA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Eq. lora_factored, LoRA term only, added onto y_in. */
int oracle_lora_apply(int64_t T, int64_t h, int64_t d, const double* x,
                      const double* y_in, int64_t n_adapters,
                      const int64_t* rank, const double* scale,
                      const int64_t* A_off, const int64_t* B_off,
                      const double* A_all, const double* B_all,
                      const int64_t* slot, double* out, int nthreads,
                      int64_t* flops_out /* nullable: + and * executed */);

/* Base forward h = xW, naive triple loop, k ascending. */
int oracle_base_forward(int64_t T, int64_t h, int64_t d, const double* x,
                        const double* W, double* out, int nthreads);

/* The padded baseline the paper rejects ("significant padding"):
 * every adapter zero-padded to r_max = max rank over adapters used in the
 * batch, then the same per-token loops with r_max.  Output must equal
 * oracle_lora_apply bit for bit (adding exact zeros).  *flops_out receives the
 * number of multiplies + adds executed by the padded loops.
 * SPEC S:219-222 (padded_oracle). */
int oracle_padded_apply(int64_t T, int64_t h, int64_t d, const double* x,
                            const double* y_in, int64_t n_adapters,
                            const int64_t* rank, const double* scale,
                            const int64_t* A_off, const int64_t* B_off,
                            const double* A_all, const double* B_all,
                            const int64_t* slot, double* out,
                            int64_t* flops_out);

#ifdef __cplusplus
}
#endif
#endif
