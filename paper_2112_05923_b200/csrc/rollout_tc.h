// rollout_tc.h -- launch descriptor of the tcgen05 fused stock rollout kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace prb {

struct TcRolloutArgs {
  const float* params;
  int a_w1, a_w2, a_w3, c_w1, c_w2, c_w3, log_std;  // flat offsets (W; b follows)
  int S, K;
  const float* shared_l1;  // [H+1][128] feat[t_h] . W1[1+K:] (actor 0-63 | critic 64-127)
  const int32_t* t_seq;    // [H+1]
  const uint8_t* done_seq; // [H]
  const double* close_tk;  // [T][K]
  const float* feat;       // [T][5K]
  double cap, max_trade, cost;
  int mt_f32;  // max_trade is an integer < 2^22: desired quantities in exact fp32 (stock::desired_qty_f32)
  int N, H;
  uint64_t seed;
  double* balance;
  int32_t* shares;   // [K][N]
  double* ep_return;
  float* obs_out;    // [N][S]
  float* b_obs;      // [H][N][1+K]
  float* b_act;      // [H][N][K]
  float* b_logp;
  float* b_val;
  float* b_rew;
  uint8_t* b_done;
  float* b_boot;
  int force_redo;   // PRB_TC_FORCE_REDO=1 (tests): every step takes the reference-division redo path
  unsigned long long* trace;  // optional clock64 phase trace of CTA 0 thread 0 (PRB_TC_TRACE), else null
};
constexpr int kTcTraceLen = 512;

size_t stock_rollout_tc_smem();
bool stock_rollout_tc_supported(int K);
void launch_stock_rollout_tc(const TcRolloutArgs& a, cudaStream_t s);
// pods x ceil(N / 128) CTAs; d_group[p] = pod p's arguments (same N, H, K for every pod)
void launch_stock_rollout_tc_group(const TcRolloutArgs* d_group, int pods, int N, int K, cudaStream_t s);

}  // namespace prb
