// pm_env.cuh -- PointMass2D transition and reset (env.hpp:84-133), shared by
// the VecEnv step kernel (env.cu) and the fused tcgen05 rollout
// (rollout_pm_tc.cu) so both produce the same bits.
//
// fp64 with explicit round-to-nearest intrinsics in the reference's operation
// order (no FMA contraction): positions, rewards, dones and step counts are
// bit-identical with the -ffp-contract=off reference build.
#pragma once
#include <cstdint>

#include "rng.cuh"

namespace prb {
namespace pm {

constexpr int kMaxSteps = 200;  // PointMass2D::spec max_episode_steps (env.hpp:117)

// std::clamp(v, lo, hi) as libstdc++ evaluates it (NaN passes through)
__device__ __forceinline__ double clamp_ref(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

// pointmass_step env.hpp:84-109.  s = (pos_x, pos_y, vel_x, vel_y, goal_x, goal_y);
// a0/a1 already clamped to the spec bounds (env.hpp:213-215).
__device__ __forceinline__ void step(const double* s, double a0, double a1, int32_t steps, double* n, double& r,
                                     bool& done) {
  const double v0 = __dadd_rn(__dmul_rn(0.9, s[2]), __dmul_rn(0.1, a0));
  const double v1 = __dadd_rn(__dmul_rn(0.9, s[3]), __dmul_rn(0.1, a1));
  n[2] = v0;
  n[3] = v1;
  n[0] = __dadd_rn(s[0], __dmul_rn(0.1, v0));
  n[1] = __dadd_rn(s[1], __dmul_rn(0.1, v1));
  n[4] = s[4];
  n[5] = s[5];
  const double action_sq = __dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1));
  const double dx = __dsub_rn(n[0], n[4]);
  const double dy = __dsub_rn(n[1], n[5]);
  const double dist = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  r = __dsub_rn(-dist, __dmul_rn(0.01, action_sq));
  const bool reached = dist < 0.05;
  if (reached) r = __dadd_rn(r, 10.0);
  done = reached || (steps + 1 >= kMaxSteps);
}

// PointMass2D::reset env.hpp:124-133: pos_x, pos_y, goal_x, goal_y ~ U(-0.4, 0.4)
// drawn in that order from the env's mt19937_64 (SoA [312][N] words); vel = 0.
__device__ __forceinline__ void reset_draws(uint64_t* mt, size_t N, int32_t& idx, double* s) {
  s[0] = mt64_uniform(mt, N, idx, -0.4, 0.4);
  s[1] = mt64_uniform(mt, N, idx, -0.4, 0.4);
  s[2] = 0.0;
  s[3] = 0.0;
  s[4] = mt64_uniform(mt, N, idx, -0.4, 0.4);
  s[5] = mt64_uniform(mt, N, idx, -0.4, 0.4);
}

}  // namespace pm
}  // namespace prb
