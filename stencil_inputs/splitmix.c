/* stencil_inputs/splitmix.c — seeded, counter-based input generator.
 *
 * This module is SHARED INPUT PLUMBING: it produces the synthetic fields that
 * both the CPU oracle (oracle/) and the CUDA path (paper_2310_01882_b200/) are
 * fed. It holds none of the method's arithmetic (no stencil, no advection):
 * only the SplitMix64 counter generator of SURVEY.md §8(d) ("Generator") and
 * an affine map of its uniform deviates onto strided buffers.
 *
 *   U01(seed, stream, idx) = (mix((seed ^ (stream*0xD1B54A32D192ED03))
 *                                 + (idx+1)*0x9E3779B97F4A7C15) >> 11) * 2^-53
 *
 * which is the (idx+1)-th output of SplitMix64 started from state
 * seed ^ (stream*0xD1B54A32D192ED03) (SPEC.md:486 `seeded:<n>`).
 * All integer arithmetic is uint64 mod 2^64. Being counter based, any element
 * of any (global) array can be generated independently, so a rank-local slab
 * gets exactly the values of the same cells of the global array.
 */
#include <stdint.h>
#include <stddef.h>

static inline uint64_t sti_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline double sti_u01_one(uint64_t state0, uint64_t idx) {
  uint64_t z = sti_mix(state0 + (idx + 1ULL) * 0x9E3779B97F4A7C15ULL);
  return (double)(z >> 11) * 0x1p-53;
}

static inline uint64_t sti_state0(uint64_t seed, uint64_t stream) {
  return seed ^ (stream * 0xD1B54A32D192ED03ULL);
}

/* Raw 64-bit output (for the generator pin G1). */
uint64_t sti_raw(uint64_t seed, uint64_t stream, uint64_t idx) {
  return sti_mix(sti_state0(seed, stream) + (idx + 1ULL) * 0x9E3779B97F4A7C15ULL);
}

double sti_u01(uint64_t seed, uint64_t stream, uint64_t idx) {
  return sti_u01_one(sti_state0(seed, stream), idx);
}

/* out[o*out_stride + i] = offset + scale * U01(seed, stream, idx_base + o*idx_stride + i)
 * for 0 <= o < n_outer, 0 <= i < n_inner. Elements of a row beyond n_inner
 * (row padding up to out_stride) are not written. Returns 0, or 1 on bad args. */
int sti_fill_affine(double* out, int64_t n_outer, int64_t n_inner, int64_t out_stride,
                    uint64_t idx_base, int64_t idx_stride, uint64_t seed, uint64_t stream,
                    double scale, double offset) {
  if (!out || n_outer < 0 || n_inner < 0 || out_stride < n_inner || idx_stride < 0) return 1;
  const uint64_t s0 = sti_state0(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t o = 0; o < n_outer; ++o) {
    double* row = out + o * out_stride;
    const uint64_t base = idx_base + (uint64_t)o * (uint64_t)idx_stride;
    for (int64_t i = 0; i < n_inner; ++i) row[i] = offset + scale * sti_u01_one(s0, base + (uint64_t)i);
  }
  return 0;
}
