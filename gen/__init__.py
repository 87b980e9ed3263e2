"""Seeded synthetic input generator shared by the oracle side and the CUDA side.

This package holds NO GEMM arithmetic. It only turns (seed, tag, i, j) counters
into the values of A, B and C_in, so that the FP64 oracle (`oracle/`) and the
CUDA path (`paper_2311_03543_b200/`) can be fed identical inputs without either
one importing the other (DESIGN.md §"Input recipe").

* `gen.inputs`   — the canonical host (numpy) generator.
* `gen/gen.cu`   — the device twin (libcompar_gen.so), which must match the host
                   generator bit for bit (checked by
                   tests/test_gpu_runtime.py::test_device_generator_matches_host_bitwise).
"""
from .inputs import (  # noqa: F401
    DIST_U, DIST_P, DIST_I, TAG_A, TAG_B, TAG_C, SEED_DATA, SEED_STREAM,
    splitmix64, counters, values_f32, values_bf16_bits, bf16_bits_to_f32,
    f32_to_bf16_bits_rne, matrix, matrix_rows, matrix_cols, matrix_entries,
)
