// ppo_tc.h -- the tensor-core PPO update (ppo_tc.cu): a group of C co-resident CTAs per learner.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace prb {

// Per learner ("chain": one ppo_update's sequence of minibatch steps).
struct PpoTcChain {
  float* params;  // the destination agent's fp32 master parameters / Adam moments (flat layout)
  float* m;
  float* v;
  int64_t* t;       // Adam step counter
  float* grads;     // [P] reduced gradient of the current step
  uint8_t* img;     // [kPpoTcImgBytes] bf16 weight image, the shared-memory layout of the MMA operands
  float* slab;      // [C][Pp] per-CTA partial gradients + loss terms
  double* stats;    // [4] sums of policy loss, value loss, entropy, accepted steps
  int32_t* status;  // [2] error code, detail
  uint32_t* sync;   // [16] zeroed before the launch: [0] barrier arrivals, [8 + c] CTA c's gate part
  const uint32_t* perm;  // injected [epochs][n] minibatch order (device indices) or null (Feistel from seed)
  uint64_t seed;
  float lr;
  // this learner's rollout buffer (time-major, index h*N + e); learners of different pods read
  // different buffers, learners of one pod the same one
  const float* obs;
  const int32_t* row;
  const float* feat;
  const float* act;
  const float* logp;
  const float* adv;
  const float* ret;
  const double* advstat;
};

struct PpoTcArgs {
  const PpoTcChain* chains;
  // nets: actor S-64-64-A, critic S-64-64-1 (flat offsets of W_l; b_l follows W_l)
  int S, A, P, Pp;
  int a_w[3], c_w[3], log_std;
  int npriv, nrest, ones_col;  // X columns: private features hi/lo [0, npriv), the rest [32, 32+nrest), ones
  // rollout buffer shape (shared by every chain of a launch; the pointers are per chain)
  int obs_mode, Sp, F;
  uint32_t N;
  // schedule
  uint32_t n, nmb;
  int bits, mb, C;
  int64_t steps;
  float clip, ent, vf;
  double b1, b2;
  float eps;
  const int2* imgpos;  // [P] weight-image position of each flat parameter (ppo_tc_image_positions)
  unsigned long long* trace;  // debug: [18] globaltimer phase marks of step 8 (null: off)
};

constexpr int kPpoTcImgBytes = 121872;
constexpr int kPpoTcMaxRows = 1024;  // 8 CTAs x 128 rows

size_t ppo_tc_smem_bytes();
// Per flat parameter: .x = byte offset of its bf16 copy in the weight image (-1: none), .y = the
// float indices of its fp32 copies in the image's fp32 block, (first | second << 16), 0xffff = none.
void ppo_tc_image_positions(const PpoTcArgs& a, int2* d_out, cudaStream_t s);
void launch_ppo_tc(const PpoTcArgs& a, int nchains, cudaStream_t s);

}  // namespace prb
