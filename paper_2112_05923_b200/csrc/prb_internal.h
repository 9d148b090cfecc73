// prb_internal.h -- internal C++ plumbing for the prb_* C ABI (include/prb.h).
//
// Error model: the reference throws nine std::runtime_error subclasses
// (common.hpp:19-71).  Every prb_* entry point runs its body under
// prb_guard(), which maps a thrown prb::Error{code} to the matching PRB_ERR_*
// code and stores the message in a thread-local slot (prb_last_error()).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <memory>
#include <vector>

#include "../../include/prb.h"

namespace prb {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

void set_last_error(int code, const std::string& msg);

template <typename F>
int guard(F&& f) {
  try {
    f();
    return PRB_OK;
  } catch (const Error& e) {
    set_last_error(e.code, e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(PRB_ERR_USAGE, e.what());
    return PRB_ERR_USAGE;
  }
}

#define PRB_CUDA(call)                                                                              \
  do {                                                                                              \
    cudaError_t err_ = (call);                                                                      \
    if (err_ != cudaSuccess)                                                                        \
      ::prb::fail(PRB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(err_) + " @" + __FILE__ + \
                                    ":" + std::to_string(__LINE__));                               \
  } while (0)

#define PRB_CHECK_LAUNCH() PRB_CUDA(cudaGetLastError())

#define PRB_REQUIRE(cond, code, msg) \
  do {                               \
    if (!(cond)) ::prb::fail(code, msg); \
  } while (0)

// Device allocation owned by a handle.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count) PRB_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
  void ensure(size_t count) {  // grow-only (keeps the allocation across calls)
    if (n < count) alloc(count);
  }
};

// Per-device opt-in to more than 48 KB of dynamic shared memory.  The
// attribute belongs to the device context, so it is set once per (kernel,
// device) -- a process driving several GPUs (one host thread per pod, the
// reference's threading model) opts in on each of them;
// thread-safe.  Call with the launching device current.
void ensure_smem_attr(const void* kernel, size_t smem_bytes);
template <typename K>
inline void ensure_smem(K* kernel, size_t smem_bytes) {
  ensure_smem_attr(reinterpret_cast<const void*>(kernel), smem_bytes);
}

// Test-only switches (prb_debug_set_option, PRB_OPT_* in prb.h); 0 unless a test set them.
int debug_option(int option);
// Developer tracing / A-B knobs: read from the environment only in a build with
// -DPRB_DEBUG_KNOBS (make NVFLAGS_EXTRA=-DPRB_DEBUG_KNOBS); nullptr otherwise.
const char* debug_env(const char* name);

uint64_t splitmix64(uint64_t x);
uint64_t derive_seed(uint64_t base, std::initializer_list<uint64_t> tags);

}  // namespace prb

// ---------------------------------------------------------------------------
// Handle structs (opaque in prb.h).
// ---------------------------------------------------------------------------

// Spin-barrier watchdog (device): a barrier still waiting 20 s after its first check aborts the
// kernel (a CUDA error on the host) instead of hanging the GPU.  Called every 1,024 polls.
__device__ __forceinline__ void barrier_watchdog(unsigned long long& t0) {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  if (t0 == 0) {
    t0 = g;
  } else if (g - t0 > 20000000000ULL) {
    asm volatile("trap;");
  }
}

struct prb_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  // pinned host staging, grown on demand (host-buffer entry points)
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* scratch = nullptr;  // device scratch, grown on demand
  size_t scratch_bytes = 0;
  unsigned int* done_counter = nullptr;  // zero between launches (last-CTA reductions reset it)
  unsigned int* last_cta_counter();
  void* pinned_staging(size_t bytes);
  void* device_scratch(size_t bytes);
  void sync();
  // Per-kernel CUDA-event timing on this stream (prb_ctx_profile_*).
  bool profiling = false;
  struct Ev {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Ev> ev_live;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[16] = {0};
  uint64_t prof_n[16] = {0};
  cudaEvent_t take_event();
};

// Makes the context's device current for the duration of an entry point and
// restores the caller's device afterwards (every launching prb_* entry opens
// one, so two contexts on two GPUs can be driven from one host thread).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const prb_ctx_s* c) {
    if (!c) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != c->device) {
      PRB_CUDA(cudaSetDevice(c->device));
      prev = cur;
    }
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};

// Kernel classes reported by prb_ctx_profile_read (index == PRB_PROF_* in prb.h).
enum { kProfPolicy = 0, kProfEnvStock = 1, kProfEnvPm = 2, kProfGae = 3, kProfPpoFwdBwd = 4, kProfPpoReduce = 5,
       kProfAdam = 6, kProfRollout = 7, kProfCount = 8 };

// RAII event pair around one launch when the context is profiling.
struct ProfScope {
  prb_ctx_s* c;
  int kind;
  cudaEvent_t a = nullptr;
  ProfScope(prb_ctx_s* ctx, int k) : c(ctx), kind(k) {
    if (c && c->profiling) {
      a = c->take_event();
      cudaEventRecord(a, c->stream);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = c->take_event();
      cudaEventRecord(b, c->stream);
      c->ev_live.push_back({kind, a, b});
    }
  }
};

struct prb_market_s {
  prb_ctx_s* ctx = nullptr;
  int K = 0;
  size_t T = 0;
  std::vector<double> close;       // [K][T] host copy (reference layout)
  std::vector<double> indicators;  // [4][K][T]
  prb::DevBuf<double> d_close_tk;  // [T][K] time-major prices for the accounting
};

enum { PRB_KIND_STOCK = 1, PRB_KIND_POINTMASS = 2 };

struct prb_vecenv_s {
  prb_ctx_s* ctx = nullptr;
  int kind = 0;
  size_t N = 0, S = 0, A = 0;
  size_t max_episode_steps = 0;
  double reward_target = 0.0;
  std::vector<double> action_low, action_high;
  bool was_reset = false;
  prb::DevBuf<float> d_obs;  // [N][S] current states (VectorizedEnvironment::states_, env.hpp:244)
  // --- stock (stock_env.hpp:135-184); lock-step: one t for all envs
  prb_market_s* market = nullptr;
  prb_stock_config cfg{};
  size_t start = 0, end = 0;
  size_t t = 0;            // uniform portfolio time index (stock_env.hpp:161)
  uint64_t step_count = 0; // uniform VecEnv step counter (env.hpp:217)
  prb::DevBuf<float> d_feat;       // [T][5K] shared obs features for this window
  prb::DevBuf<double> d_balance;   // [N]
  prb::DevBuf<int32_t> d_shares;   // [K][N]
  prb::DevBuf<double> d_ep_return; // [N]
  // --- point mass (env.hpp:111-146)
  prb::DevBuf<double> d_pm_state;   // [6][N]
  prb::DevBuf<int32_t> d_pm_steps;  // [N]
  prb::DevBuf<uint64_t> d_mt;       // [312][N] per-env mt19937_64 words
  prb::DevBuf<int32_t> d_mt_idx;    // [N]
  // scratch for the host-buffer step
  prb::DevBuf<float> d_act_scratch, d_rew_scratch, d_term_scratch;
  prb::DevBuf<uint8_t> d_done_scratch;
  prb::DevBuf<double> d_tret_scratch;
  prb::DevBuf<int32_t> d_tlen_scratch;
};

// Device parameter blob in the reference's canonical flat layout
// (artifact.hpp:35-51): actor layers (W [in x out] row-major, then b),
// log_std[A], critic layers.  fp32 master weights + Adam m/v (nn.hpp:144-152).
struct prb_agent_s {
  prb_ctx_s* ctx = nullptr;
  size_t S = 0, A = 0;
  std::vector<size_t> hidden;
  std::vector<size_t> adims, cdims;  // actor/critic layer dims
  size_t P = 0, Pa = 0, Pc = 0;      // total, actor-MLP, critic-MLP param counts
  std::vector<size_t> aoff, coff;    // per-layer W offsets into the flat blob
  double lr = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  prb::DevBuf<float> d_params, d_m, d_v, d_grads;
  prb::DevBuf<int64_t> d_t;          // Adam step counter (device-resident)
  prb::DevBuf<int32_t> d_status;     // [0]=error code raised on device, [1]=detail
  std::shared_ptr<void> ppo_ws;      // ppo.cu workspace, kept across prb_ppo_update calls
  int ppo_mode = 0;                  // prb_agent_set_ppo_mode: 0 fp32 SIMT (default), 1 tensor cores where supported
};

// Device TransitionBuffer (buffer.hpp:27-135), TIME-MAJOR: transition
// (env e, step h) lives at index h*N + e.  The reference's env-major index is
// e*H + h (pod.hpp:89-94); prb_rollout_* host transfers convert.
struct prb_rollout_s {
  prb_ctx_s* ctx = nullptr;
  size_t N = 0, H = 0, S = 0, A = 0;
  int obs_mode = 0;  // 0 = full rows [cap][S]; 1 = stock compact: private [cap][1+K] + shared feature row per step
  size_t Sp = 0;     // stored obs floats per transition
  int K = 0;
  prb::DevBuf<float> d_obs;        // [cap][Sp]
  prb::DevBuf<int32_t> d_row;      // [H] shared feature row (stock compact)
  const float* d_feat = nullptr;   // [T][5K] feature table of the producing env (compact mode)
  prb::DevBuf<float> d_act;        // [cap][A]
  prb::DevBuf<float> d_logp, d_rew, d_val, d_adv, d_ret;  // [cap]
  prb::DevBuf<uint8_t> d_done;     // [cap]
  prb::DevBuf<float> d_boot;       // [N] bootstrap V(s_H)
  prb::DevBuf<uint8_t> d_pack;     // bf16 weight chunks of the PointMass 3x256 tcgen05 rollout
  prb::DevBuf<double> d_advstat;   // mean, denom of the advantages (ppo.hpp:234-242)
  // grouped (multi-pod) tcgen05 collect: this rollout's step schedule and shared first-layer term
  prb::DevBuf<float> d_sl;         // [H+1][128]
  prb::DevBuf<int32_t> d_tseq;     // [H+1]
  prb::DevBuf<uint8_t> d_dseq;     // [H]
  bool gae_valid = false;
  bool normalized = true;
  bool full = false;
  int mode = 2;  // prb_rollout_set_mode: 0 per-step kernels, 1 fused fp32 SIMT, 2 fused tcgen05 (default)
};
