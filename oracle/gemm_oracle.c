/*
 * oracle/gemm_oracle.c — FP64 reference GEMM.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2311_03543_b200/, include/compar.h) never links, includes or calls it,
 * and this file includes nothing from the product tree.
 *
 * What it computes (the plain definition):
 *
 *     C_out[i][j] = alpha * sum_{k=0}^{K-1} A[i][k] * B[k][j]  +  beta * C_in[i][j]
 *
 * for 0 <= i < M, 0 <= j < N — the matrix-multiply component ("mmul") of
 * PAPER.md P:76-80 [§2.1, Listing 3 text] and its BLAS/cuBLAS variants in
 * P:201-205 [Table 2, "Matrix multiply: BLAS, OMP, CUDA, CUBLAS"], read with
 * xGEMM semantics C = alpha*A*B + beta*C (BASELINE.json north_star; DESIGN.md
 * reading R1).  BLAS quick-return rules (reading R3):
 *   * beta == 0  -> C_in is not read (NaN/Inf in C_in do not propagate);
 *   * alpha == 0 -> A and B are not read; C_out = beta * C_in;
 *   * K == 0     -> the sum is empty (0).
 *
 * How: plain triple loop in the order i, k, j, so each C element is summed in
 * increasing k; FP64 accumulation; row-major operands with explicit leading
 * dimensions; OpenMP over rows only (each row is independent, so the result
 * does not depend on the thread count).  Built with -O2 -ffp-contract=off and
 * no -march / fast-math so it is host-independent.  Inputs arrive already
 * widened (exactly) to FP64 by oracle/gemm.py.
 *
 * parity pins: tests/test_oracle_pins.py (worked examples, closed forms,
 * exact-rational brute force, numpy float64 cross-check, BLAS special cases).
 */
#include <stddef.h>

void compar_oracle_gemm(long M, long N, long K, double alpha,
                        const double *A, long lda,
                        const double *B, long ldb,
                        double beta, const double *C_in, long ldc_in,
                        double *C_out, long ldc_out)
{
    long i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < M; ++i) {
        double *c = C_out + i * ldc_out;
        long j, k;
        for (j = 0; j < N; ++j)
            c[j] = 0.0;
        if (alpha != 0.0) {
            for (k = 0; k < K; ++k) {
                const double a = A[i * lda + k];
                const double *b = B + k * ldb;
                for (j = 0; j < N; ++j)
                    c[j] += a * b[j];
            }
        }
        for (j = 0; j < N; ++j) {
            const double acc = alpha * c[j];
            c[j] = (beta == 0.0) ? acc : acc + beta * C_in[i * ldc_in + j];
        }
    }
}

/* Number of OpenMP threads the oracle will use (reported as cpu_baseline.cores). */
int compar_oracle_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Set the OpenMP thread count for later calls (the bench's 1-thread vs all-threads timing of the
 * oracle); rows are independent, so results do not depend on it. */
void compar_oracle_set_threads(int n)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
