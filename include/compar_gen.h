/*
 * compar_gen.h — device twin of the seeded input generator (gen/gen.cu -> gen/libcompar_gen.so).
 *
 * Not part of the GEMM method: it only materialises the synthetic inputs of SURVEY.md §8(d)
 * ("Inputs") on the GPU so that full-size workloads (e.g. 32768^3) need no host->device copy
 * of generated data.  It implements the same counter-based recipe as the canonical host
 * generator gen/inputs.py and must match it bit for bit
 * (tests/test_gpu_runtime.py::test_device_generator_matches_host_bitwise):
 *
 *     h = splitmix64(seed ^ (tag << 56) ^ (i << 28) ^ j)        (i, j) = LOGICAL row, column
 *     U = ((h >> 40) - 2^23) * 2^-23,  P = (h >> 40) * 2^-24,  I = h mod 5 - 2
 *     BF16 = round-to-nearest-even of the FP32 value.
 *
 * Neither the oracle nor the product library links this; tests and bench.py call it.
 */
#ifndef COMPAR_GEN_H
#define COMPAR_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Fill a rows x cols block of a LOGICAL matrix, whose top-left element is logical (row0, col0),
 * into device memory `dst` (row pitch `ld` elements) — e.g. one rank's row panel of A.
 *   dtype: 0 = FP32, 1 = BF16 bit patterns;  dist: 0 = U, 1 = P, 2 = I;
 *   transposed = 1 stores logical (i, j) at dst[j * ld + i] (e.g. B^T for transB; ld >= rows),
 *   else at dst[i * ld + j] (ld >= cols).
 *   stream: cudaStream_t or NULL.  Asynchronous.  Returns 0 on success, else a cudaError_t
 *   value (1 = invalid argument). */
int compar_gen_fill(void *dst, int dtype, int64_t rows, int64_t cols, int64_t ld, int64_t row0, int64_t col0,
                    uint64_t seed, int tag, int dist, int transposed, void *stream);

#ifdef __cplusplus
}
#endif
#endif
