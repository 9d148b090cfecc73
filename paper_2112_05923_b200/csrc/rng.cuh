// rng.cuh -- counter-based and reference-exact random streams on device.
//
//  * splitmix64 / derive_seed: common.hpp:79-93, integer-exact.
//  * mt19937_64 + libstdc++ uniform_real_distribution<double>: the per-env
//    reset stream of VectorizedEnvironment (env.hpp:186-194) and
//    PointMass2D::reset (env.hpp:124-133).  Reproduced bit-exactly so device
//    resets equal the reference's (u = double(x)/2^64, then u*(b-a)+a with
//    no FMA contraction, as the -ffp-contract=off reference build).
//  * Philox4x32-10: policy noise / permutations / mutation (the reference's
//    std::normal_distribution draws are not reproducible in parallel; the
//    checker regenerates these draws with the same Philox, oracle/*.c).
#pragma once
#include <cstdint>

namespace prb {

__host__ __device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// derive_seed(base, a, b) (common.hpp:88-93)
__host__ __device__ __forceinline__ uint64_t derive_seed2(uint64_t base, uint64_t a, uint64_t b) {
  uint64_t s = splitmix64_d(base);
  s = splitmix64_d(s ^ splitmix64_d(a));
  s = splitmix64_d(s ^ splitmix64_d(b));
  return s;
}

struct Philox4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ Philox4 philox4x32_10(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1,
                                                          uint32_t c2, uint32_t c3) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return Philox4{c0, c1, c2, c3};
}

// Two unit normals from two 32-bit draws (Box-Muller, fp32).  The top 23 bits of each draw become
// the mantissa of a float in [1, 2) (one LEA.HI each, no int->float conversion); u1 = 2 - that is
// in (0, 1] (>= 2^-23, so the log never sees 0 or a denormal), and sin/cos take 2*pi*[1, 2), the
// same angles as [0, 1).  SFU forms (MUFU.LG2 / SQRT / SIN / COS): sampling noise needs ~1e-6,
// not correct rounding.
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
  const float u1 = 2.0f - __uint_as_float(0x3F800000u | (a >> 9));
  const float x2 = __uint_as_float(0x3F800000u | (b >> 9));
  float lg, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(u1));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-1.3862943611198906f * lg));  // sqrt(-2 ln u1)
  float s, c;
  __sincosf(6.2831853071795865f * x2, &s, &c);
  return make_float2(r * c, r * s);
}

// ---- mt19937_64, state SoA [312][N] + idx[N] --------------------------------
constexpr int kMtN = 312;

__device__ __forceinline__ void mt64_seed(uint64_t* mt, size_t stride, uint64_t seed) {
  uint64_t prev = seed;
  mt[0] = prev;
  for (int i = 1; i < kMtN; ++i) {
    prev = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)i;
    mt[(size_t)i * stride] = prev;
  }
}

__device__ __forceinline__ void mt64_twist(uint64_t* mt, size_t stride) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  uint64_t cur = mt[0];
  for (int i = 0; i < kMtN; ++i) {
    // the last word pairs with the already-regenerated mt[0] (libstdc++ _M_gen_rand)
    const uint64_t nxt = mt[(size_t)((i + 1) % kMtN) * stride];
    // mt[(i+156)%312]: for i >= 156 this is an already-updated word (as in the reference loop)
    const uint64_t far = mt[(size_t)((i + 156) % kMtN) * stride];
    const uint64_t y = (cur & upper) | (nxt & lower);
    uint64_t v = far ^ (y >> 1);
    if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
    mt[(size_t)i * stride] = v;
    cur = nxt;
  }
}

__device__ __forceinline__ uint64_t mt64_next(uint64_t* mt, size_t stride, int32_t& idx) {
  if (idx >= kMtN) {
    mt64_twist(mt, stride);
    idx = 0;
  }
  uint64_t x = mt[(size_t)idx * stride];
  ++idx;
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

// uniform_real_distribution<double>(a, b) over generate_canonical<double,53>
__device__ __forceinline__ double mt64_uniform(uint64_t* mt, size_t stride, int32_t& idx, double a, double b) {
  double u = __dmul_rn(__ull2double_rn(mt64_next(mt, stride, idx)), 5.421010862427522170037264e-20);  // 2^-64
  if (u >= 1.0) u = 0.99999999999999988898;  // nextafter(1, 0)
  return __dadd_rn(__dmul_rn(u, __dsub_rn(b, a)), a);
}

}  // namespace prb
