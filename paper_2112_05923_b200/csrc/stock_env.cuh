// stock_env.cuh -- shared device pieces of stock_env_step (stock_env.hpp:55-103).
#pragma once

namespace prb {
namespace stock {

// Buy quantity  min(desired, max(floor(balance / (price * (1 + cost))), 0))
// (stock_env.hpp:91-97), bit-identical to the reference, with the fp64
// division skipped when it cannot matter: if the EXACT product desired * pc
// is <= balance (its sign is that of the single-rounding FMA residual), the
// exact quotient is >= desired, so is its rounding (desired is a double), and
// floor() of it; the result is then `desired` itself.  Only cash-limited buys
// pay for __ddiv_rn, which is the long pole of the per-env dependency chain.
// The cash-limited slow path is out of line: inlining __ddiv_rn's sequence once
// per asset of an unrolled K-loop bloats the kernels past the instruction cache.
static __device__ __noinline__ double buy_qty_limited(double desired, double balance, double pc) {
  const double affordable = floor(__ddiv_rn(balance, pc));
  const double floor0 = (affordable < 0.0) ? 0.0 : affordable;  // std::max(affordable, 0.0)
  return (floor0 < desired) ? floor0 : desired;                  // std::min(desired, .)
}

// Largest double below 1.  If pc * kBelowOne >= balance (exact sign of the single-rounding
// FMA residual), the exact quotient balance/pc is <= kBelowOne, so its rounding is < 1 and
// floor() gives 0: the cash-limited buy of an env that cannot afford one share, decided
// without the fp64 division (the common case once a portfolio's cash is spent).
constexpr double kBelowOne = 0.99999999999999988898;  // 1 - 2^-53

__device__ __forceinline__ bool cannot_afford_one(double balance, double pc) {
  return __fma_rn(pc, kBelowOne, -balance) >= 0.0;
}

__device__ __forceinline__ double buy_qty(double desired, double balance, double pc) {
  if (__fma_rn(desired, pc, -balance) <= 0.0) return desired;
  if (cannot_afford_one(balance, pc)) return 0.0;
  return buy_qty_limited(desired, balance, pc);
}

}  // namespace stock
}  // namespace prb
