// Device realizations of the reference's draw contract (rng.hpp:17-55,
// sketch.cpp:62-79, 94-95, 119-124), bit-exact for every integer draw.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rpb {

enum class WordMode : int { Raw = 0, Uniform01 = 1, Sign = 2 };

// count outputs of SeededRng(seed) after discarding `skip`: raw next_u64,
// uniform01 or sign(), written to d_out (uint64_t* or double*).
void draw_words(uint64_t seed, uint64_t skip, int64_t count, WordMode mode, void* d_out,
                cudaStream_t stream);

// count consecutive uniform_index(bound) draws (rejection sampling honoured).
void draw_uniform_index(uint64_t seed, uint64_t bound, int64_t count, uint64_t* d_out,
                        cudaStream_t stream);

// Gaussian rows: normals of the SeededRng(seed) normal() stream at indices
// [cursor_r, cursor_r + J) for each of R rows, times `scale`, written row-major
// (out[r * ld + j]).  `d_states` holds, per row, the window at u64 offset
// 2*floor(cursor_r/2); on return the states and cursors are advanced by J.
struct GaussRows {
  int64_t rows = 0;
  uint64_t* d_states = nullptr;  // rows x 312
  int64_t* d_cursor = nullptr;   // rows
};
// Initializes states/cursors for rows whose first normal index is first + r * stride.
void gauss_rows_init(uint64_t seed, int64_t rows, int64_t first, int64_t stride, GaussRows& g,
                     cudaStream_t stream);
void gauss_rows_next(GaussRows& g, int64_t J, double scale, double* d_out, int64_t ld,
                     cudaStream_t stream);

// Normals [first, first + count) of the SeededRng(seed) normal() stream
// (first even), times `scale`, contiguous in d_out: a Gaussian sketch whose
// rows are consecutive stretches of the stream (S = m x n, row stride n) is
// one such stream -- a handful of segment jumps instead of one per row.
void draw_gauss_stream(uint64_t seed, int64_t first, int64_t count, double scale, double* d_out,
                       cudaStream_t stream);

// CountSketch / SJLT draws for the whole stream (sketch.cpp:119-124):
// h[b * n + j] (int32) and sgn[b * n + j] = sign() * entry.
void draw_count(uint64_t seed, int64_t n, int64_t rows_per_block, int blocks, double entry,
                int32_t* d_h, double* d_sgn, cudaStream_t stream);

// SRHT draws (sketch.cpp:62-79): n signs, then m partial Fisher-Yates rows.
void draw_srht(uint64_t seed, int64_t n, int64_t m, double* d_signs, int64_t* d_rows,
               cudaStream_t stream);

}  // namespace rpb
