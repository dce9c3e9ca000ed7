// hash.cuh — counter-based hashes of the synthetic-input generators (synth*.cu).
// Restated bit-for-bit in numpy by oracle/spmv_entropy_oracle.py (hash3).
#pragma once
#include <stdint.h>

namespace sme {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return mix64(seed * 0x9E3779B97F4A7C15ull + mix64(a * 0xD1B54A32D192ED03ull + b + 0x632BE59BD9B4E019ull));
}
__host__ __device__ __forceinline__ double unit_pm1(uint64_t h) {  // U[-1, 1), exact in numpy too
  return (double)(h >> 11) * 0x1p-52 - 1.0;
}
__host__ __device__ __forceinline__ double unit01(uint64_t h) {  // U[0, 1)
  return (double)(h >> 11) * 0x1p-53;
}
constexpr uint64_t VAL_SALT = 0x5DEECE66Dull;

}  // namespace sme
