// Counter-addressable std::mt19937_64 for the device.
//
// The reference draws every sketch from one std::mt19937_64 stream
// (rng.hpp:17-19, 59), consumed strictly in order (sketch.cpp:62-79, 94-95,
// 119-124).  To generate that stream in parallel we jump the generator to
// arbitrary output offsets with the GF(2) characteristic polynomial phi of the
// state transition T (degree 19937): the window W_{q+J} = p(T) W_q where
// p = x^J mod phi.  phi is recovered once per process by Berlekamp-Massey on
// the generator's own output and verified by a jump self-check.
//
// Conventions: X_t is the MT word sequence (X_0..X_311 = seeded array,
// X_{t+312} = X_{t+156} ^ twist(X_t, X_{t+1})); output q is temper(X_{312+q});
// the "state at output offset q" is the 312-word window W_q = X_q..X_{q+311}.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace rpb {
namespace mt {

constexpr int kN = 312;
constexpr int kM = 156;
constexpr int kDeg = 19937;
constexpr int kPolyWords = (kDeg + 63) / 64;  // 312
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLower = 0x000000007FFFFFFFULL;

using Poly = std::vector<uint64_t>;

// Seeded window W_0 (std::mt19937_64 seeding, [rand.eng.mers]).
void seed_window(uint64_t seed, uint64_t out[kN]);

// x^e mod phi (cached for repeated exponents).
Poly xpow(uint64_t e);

// Host reference jump: out = p(T) in.  Used by the self-check and tests.
void host_jump(const uint64_t in[kN], const Poly& p, uint64_t out[kN]);

// Host reference: first `count` outputs starting at output offset `skip`.
void host_outputs(uint64_t seed, uint64_t skip, int64_t count, uint64_t* out);

// Process-wide init (phi, Barrett constant, x^(2^i) table, self-check).
// Returns the time spent in milliseconds the first time, 0 afterwards.
double init_tables();

// Device side ---------------------------------------------------------------

// Computes the windows at output offsets `offsets[r]` (r < R) of the stream of
// `seed` into d_states (R x 312 words, device).  Uses a doubling schedule: row
// r > 0 jumps from row r - 2^floor(log2 r); the distinct differences are turned
// into jump polynomials on the host (cached), so arithmetic progressions cost
// one polynomial per level.  Returns the number of kernel launches.
int states_at(uint64_t seed, const std::vector<uint64_t>& offsets, uint64_t* d_states,
              cudaStream_t stream);

}  // namespace mt
}  // namespace rpb
