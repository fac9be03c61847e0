// Device generator of synthetic Balding-Nichols genotypes (BASELINE.json
// configs). Counter-based: every draw is a hash of (seed, marker, sample,
// stream), so any shard or sub-block regenerates identically on CPU and GPU.
// The draw definition is shared with the CPU oracle
// (oracle/gkb_oracle.c:orc_synth_bed); products and sums use explicit
// round-to-nearest intrinsics so no FMA contraction changes a frequency.
// Frequencies (Beta / Dirichlet draws) are made on the host and passed in.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace gkb {
namespace dev {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u53(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
__device__ __forceinline__ uint64_t marker_key(uint64_t seed, int64_t j) {
  return mix64(seed * 0x9E3779B97F4A7C15ULL + (uint64_t)j + 1ULL);
}
__device__ __forceinline__ uint64_t cell_key(uint64_t mk, int64_t i) {
  return mix64(mk ^ ((uint64_t)i * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
}

__device__ double sample_freq(const SynthDev& s, int64_t j, int64_t i) {
  if (s.pop) return s.freq[(int64_t)s.pop[i] * s.p + j];
  double acc = 0.0;
  for (int k = 0; k < s.npop; ++k)
    acc = __dadd_rn(acc, __dmul_rn(s.admix[i * s.npop + k], s.freq[(int64_t)k * s.p + j]));
  return acc;
}

__device__ int draw_dosage(const SynthDev& s, uint64_t mk, int64_t j, int64_t i) {
  const uint64_t h = cell_key(mk, i);
  const double f = sample_freq(s, j, i);
  int d = (u53(mix64(h + 1)) < f) + (u53(mix64(h + 2)) < f);
  if (s.copy_from && s.copy_from[i] >= 0 && u53(mix64(h + 4)) < s.copy_prob) {
    const int64_t a = s.copy_from[i];
    const uint64_t ha = cell_key(mk, a);
    const double fa = sample_freq(s, j, a);
    d = (u53(mix64(ha + 1)) < fa) + (u53(mix64(ha + 2)) < fa);
  }
  if (s.missing_rate > 0.0 && u53(mix64(h + 3)) < s.missing_rate) return 3;
  return d;
}

// thread per (row, byte): 4 samples
__global__ void k_synth_bed(SynthDev s, int64_t j0, int64_t rows, uint8_t* __restrict__ out) {
  const int64_t stride = (s.n + 3) / 4;
  const int64_t total = rows * stride;
  const uint8_t kDosageToCode[4] = {3, 2, 0, 1};
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = idx / stride, b = idx - rr * stride;
    const int64_t j = j0 + rr;
    const uint64_t mk = marker_key(s.seed, j);
    uint32_t byte = 0;
    for (int t = 0; t < 4; ++t) {
      const int64_t i = 4 * b + t;
      if (i >= s.n) break;
      byte |= (uint32_t)kDosageToCode[draw_dosage(s, mk, j, i)] << (2 * t);
    }
    out[idx] = (uint8_t)byte;
  }
}

}  // namespace

void synth_bed(const SynthDev& sp, int64_t j0, int64_t rows, uint8_t* out, cudaStream_t s) {
  const int64_t total = rows * ((sp.n + 3) / 4);
  if (total == 0) return;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_synth_bed<<<(unsigned)g, 256, 0, s>>>(sp, j0, rows, out);
}

}  // namespace dev
}  // namespace gkb
