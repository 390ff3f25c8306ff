// Test helper (built by tests/test_gpu_division.py): compares div_by(a, b,
// rcp_div(b)) with the device's own a / b on pseudo-random operand bit
// patterns (all exponents, signs, NaN/Inf/subnormal included) and on
// normal-range operands; counts bitwise mismatches.
#include <cstdint>

#include "physics.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void k_div_check(uint64_t n, uint64_t seed, int mode, unsigned long long* bad) {
  unsigned long long local = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t ra = mix(seed ^ (2 * i)), rb = mix(seed ^ (2 * i + 1));
    if (mode == 1) {  // normal range around 1 (exponents 1023 +- 64)
      ra = (ra & 0x800fffffffffffffull) | ((uint64_t)(1023 - 64 + (ra >> 52) % 128) << 52);
      rb = (rb & 0x800fffffffffffffull) | ((uint64_t)(1023 - 64 + (rb >> 52) % 128) << 52);
    } else if (mode == 2) {  // near-tie quotients: b from a small integer grid
      rb = __double_as_longlong((double)(1 + (rb % 4096)));
    }
    const double a = __longlong_as_double((long long)ra), b = __longlong_as_double((long long)rb);
    const double y = tafv::rcp_div(b);
    const double q = tafv::div_by(a, b, y);
    const double ref = a / b;
    const bool same = __double_as_longlong(q) == __double_as_longlong(ref) || (ref != ref && q != q);
    local += same ? 0 : 1;
  }
  if (local) atomicAdd(bad, local);
}

extern "C" int div_check(unsigned long long n, unsigned long long seed, int mode, unsigned long long* out) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof *d) != cudaSuccess) return 1;
  cudaMemset(d, 0, sizeof *d);
  k_div_check<<<148 * 16, 256>>>(n, seed, mode, d);
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  cudaMemcpy(out, d, sizeof *d, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return 0;
}
