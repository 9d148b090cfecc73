// rollout_pm_tc.h -- launch descriptor of the tcgen05 PointMass 3x256 rollout.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace prb {

constexpr int kPmChunkK = 32;  // K per streamed weight chunk of the 256x256 layers (16 or 32)
// bf16 weight chunks of both nets: per net W1 | 256/kPmChunkK chunks each of W2, W3 | W4
constexpr uint32_t kPmPackBytes = 2u * (2 + 2 * (256 / kPmChunkK)) * (256u * kPmChunkK * 2);

struct PmPackOffsets {
  int S, A;                // 6, 2
  int a_w[4], c_w[4];      // flat W offsets of the 4 layers (bias follows each W)
  int log_std;
};

struct PmTcArgs {
  CUtensorMap pack_map; // the pack as a 2-D bf16 tensor [kPmPackBytes/256][128], box [16][128] (CTA-pair kernel)
  const uint8_t* pack;  // kPmPackBytes, from launch_pm_pack
  const float* params;
  PmPackOffsets o;
  int N, H;
  uint64_t seed;
  double* st;        // [6][N]
  int32_t* steps;    // [N]
  double* ep_return; // [N]
  uint64_t* mt;      // [312][N]
  int32_t* mt_idx;   // [N]
  float* obs_out;    // [N][6]
  float* b_obs;      // [H][N][6]
  float* b_act;      // [H][N][2]
  float* b_logp;
  float* b_val;
  float* b_rew;
  uint8_t* b_done;
  float* b_boot;
  unsigned long long* trace;  // optional [4][kPmTraceLen] clock64 events of CTA 0 (PRB_PM_TRACE), else null
};
constexpr int kPmTraceLen = 512;

size_t pm_rollout_tc_smem();
void launch_pm_pack(const float* params, const PmPackOffsets& o, uint8_t* pack, cudaStream_t s);
void launch_pm_rollout_tc(const PmTcArgs& a, int num_sms, cudaStream_t s);

}  // namespace prb
