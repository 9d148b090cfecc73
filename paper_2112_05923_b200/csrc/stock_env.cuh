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

// ---- conversion- and division-free pieces of the fused rollout's env step ----
// The fp64 <-> int conversions (I2F.F64 / F2I.F64) and __ddiv_rn run on the
// quarter-rate XU pipe and sit on the per-env dependency chain through the
// balance; these restatements use only the fp32 / fp64 FMA pipes and integer
// ops and are bit-identical to the reference expressions they replace.

// (double)i for any int32, exact: the double 2^52 + 2^31 + i has low word i + 2^31.
__device__ __forceinline__ double i2d_exact(int32_t i) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)((uint32_t)i ^ 0x80000000u)), 4503601774854144.0);
}

// desired = trunc(clamp(a, -1, 1) * max_trade) (stock_env.hpp:83-87) for an fp32 action and an
// integer-valued max_trade < 2^22 (mt as a float and as mti, both exact).  In fp64 the product
// of a 24-bit action and a <= 22-bit integer is exact, so the reference truncates the EXACT
// product x.  RZ(x) (the fp32 product rounded toward zero) has the same truncation: no integer
// lies strictly between x and RZ(x), every integer below 2^24 being a float.  The clamp of the
// action to [-1, 1] is then the clamp of the integer to [-mti, mti] (RZ is monotone and mt is
// exact); cvt.rzi maps NaN to 0 (the reference: a NaN desired is neither < 0 nor > 0, no
// trade) and saturates infinities.
__device__ __forceinline__ int32_t desired_qty_f32(float a, float mt, int32_t mti) {
  const int32_t d = __float2int_rz(__fmul_rz(a, mt));
  return min(max(d, -mti), mti);
}

// Per step and asset, shared by every env of the VecEnv (lock-step t): pc = price * (1 + c),
// inv = RN(1 / pc), thr = pc * 2^-50.
struct BuyPrice {
  double pc, inv, thr;
};

__device__ __forceinline__ BuyPrice buy_price(double price, double cost_rate) {
  BuyPrice b;
  b.pc = __dmul_rn(price, __dadd_rn(1.0, cost_rate));
  b.inv = __drcp_rn(b.pc);
  b.thr = __dmul_rn(b.pc, 0x1p-50);
  return b;
}

// Buy quantity min(desired, max(floor(RN(balance / pc)), 0)) (stock_env.hpp:91-97) as int32,
// without the division.  qa = RN(balance · inv) is within 2^-51·q of q = balance / pc (two
// roundings), RN(q) within 2^-53·q.  For 0 < qa < 2^31 those are < 2^-19.7, so when the fraction
// of qa is more than 2^-19 away from both integers, q and RN(q) lie strictly inside
// (floor(qa), floor(qa) + 1) and floor(RN(q)) = floor(qa) = n.  n comes from the 2^52-biased
// round-down add; its int32 value is the low word.  Any lane outside that certificate (quotient
// within 2^-19 of an integer, balance <= 0, absurd cash) takes the reference's own division; the
// warp-uniform vote keeps that path out of line.  Non-buys (desired <= 0) give 0.
__device__ __forceinline__ int32_t buy_qty_i32(int32_t di, double balance, const BuyPrice& b) {
  const double qa = __dmul_rn(balance, b.inv);
  const double t = __dadd_rd(qa, 0x1p52);
  const double frac = __dsub_rn(qa, __dsub_rn(t, 0x1p52));
  const bool ok = (fabs(__dsub_rn(frac, 0.5)) < 0.5 - 0x1p-19) && (fabs(__dsub_rn(qa, 0x1p30)) < 0x1p30);
  int32_t n = __double2loint(t);
  if (__any_sync(0xffffffffu, !ok)) {
    if (!ok) n = (int32_t)buy_qty_limited((double)di, balance, b.pc);
  }
  return max(min(n, di), 0);
}

// buy_qty_i32 without the vote: the certificate failure is accumulated in `bad` and the caller
// redoes the whole trade sequence with the reference's division when any lane of the warp saw
// one (rollout_tc.cu); the returned quantity is then discarded.
__device__ __forceinline__ int32_t buy_qty_i32_spec(int32_t di, double balance, const BuyPrice& b, bool& bad) {
  const double qa = __dmul_rn(balance, b.inv);
  const double t = __dadd_rd(qa, 0x1p52);
  const double frac = __dsub_rn(qa, __dsub_rn(t, 0x1p52));
  bad |= !((fabs(__dsub_rn(frac, 0.5)) < 0.5 - 0x1p-19) && (fabs(__dsub_rn(qa, 0x1p30)) < 0x1p30));
  return max(min((int32_t)__double2loint(t), di), 0);
}

}  // namespace stock
}  // namespace prb
