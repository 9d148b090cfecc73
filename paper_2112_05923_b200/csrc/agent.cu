// agent.cu -- the device AgentArtifact (artifact.hpp:23-86): flat fp32
// parameter blob in the reference's canonical order, Adam state (nn.hpp:144-182),
// learner fusion (pod.hpp:141-172), leaderboard ranking (tournament.hpp:104-119)
// and the generator's mutation (tournament.hpp:149-159).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "mlp_simt.cuh"
#include "prb_internal.h"
#include "rng.cuh"

using namespace prb;

namespace {

void layout(prb_agent_s* a) {
  a->adims.clear();
  a->cdims.clear();
  a->adims.push_back(a->S);
  a->cdims.push_back(a->S);
  for (size_t h : a->hidden) {
    a->adims.push_back(h);
    a->cdims.push_back(h);
  }
  a->adims.push_back(a->A);
  a->cdims.push_back(1);
  size_t off = 0;
  a->aoff.clear();
  for (size_t i = 0; i + 1 < a->adims.size(); ++i) {
    a->aoff.push_back(off);
    off += a->adims[i] * a->adims[i + 1] + a->adims[i + 1];
  }
  a->Pa = off;
  off += a->A;  // log_std
  a->coff.clear();
  for (size_t i = 0; i + 1 < a->cdims.size(); ++i) {
    a->coff.push_back(off);
    off += a->cdims[i] * a->cdims[i + 1] + a->cdims[i + 1];
  }
  a->P = off;
  a->Pc = a->P - a->Pa - a->A;
}

// adam_step nn.hpp:164-182 on device; gate[0] != 0 aborts without touching state.
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, size_t n, const int64_t* __restrict__ t_dev,
                            const int32_t* __restrict__ gate, float lr, double b1d, double b2d, float eps) {
  if (gate && gate[0] != 0) return;
  const int64_t t = *t_dev;  // already advanced by the producer of g
  const double bc1 = 1.0 - pow(b1d, (double)t);
  const double bc2 = 1.0 - pow(b2d, (double)t);
  const float ibc1 = (float)(1.0 / bc1), ibc2 = (float)(1.0 / bc2);
  // constants rounded once from fp64 (1 - beta2 in fp32 arithmetic would be off by 1e-5 relative)
  const float b1 = (float)b1d, b2 = (float)b2d, omb1 = (float)(1.0 - b1d), omb2 = (float)(1.0 - b2d);
  auto upd = [&](float gi, float& mi, float& vi, float& pi) {
    mi = b1 * mi + omb1 * gi;
    vi = b2 * vi + omb2 * gi * gi;
    pi -= lr * (mi * ibc1) / (sqrtf(vi * ibc2) + eps);
  };
  const size_t tid0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  size_t n4 = 0;
  if (((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(m) |
        reinterpret_cast<uintptr_t>(v)) & 15) == 0) {  // 16-byte streams (same arithmetic per element)
    n4 = n / 4;
    float4* p4 = reinterpret_cast<float4*>(p);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    float4* m4 = reinterpret_cast<float4*>(m);
    float4* v4 = reinterpret_cast<float4*>(v);
    for (size_t i = tid0; i < n4; i += stride) {
      const float4 gg = g4[i];
      float4 mm = m4[i], vv = v4[i], pp = p4[i];
      upd(gg.x, mm.x, vv.x, pp.x);
      upd(gg.y, mm.y, vv.y, pp.y);
      upd(gg.z, mm.z, vv.z, pp.z);
      upd(gg.w, mm.w, vv.w, pp.w);
      m4[i] = mm;
      v4[i] = vv;
      p4[i] = pp;
    }
  }
  for (size_t i = 4 * n4 + tid0; i < n; i += stride) {
    float mi = m[i], vi = v[i], pi = p[i];
    upd(g[i], mi, vi, pi);
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
  }
}

// Grid-wide finite check of the gradients (nn.hpp:169-171: reject before touching state).
// status[2] counts finished CTAs, status[3] collects the non-finite flag; the last CTA
// publishes the verdict (status[0..1]) and advances t on success, then re-arms [2] and [3].
__global__ void finite_check_kernel(const float* __restrict__ g, size_t n, int32_t* status, int64_t* t_dev) {
  int local = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    local |= !isfinite(g[i]);
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(&status[3], 1);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&status[2], 1) == (int)gridDim.x - 1) {
      __threadfence();
      const int bad = atomicExch(&status[3], 0);
      status[2] = 0;
      if (bad) {
        status[0] = PRB_ERR_NUMERIC;
        status[1] = 1;  // adam_step: non-finite gradient
      } else {
        status[0] = 0;
        *t_dev += 1;
      }
    }
  }
}

// params, m and v of L agents (src: L param pointers, then L m, then L v) -> their means, one
// pass; element i of every output is written after every input's element i is read, so an
// output may alias an input.  Block 0 also sets t = max of the L counters (pod.hpp:149-171).
__global__ void fuse_kernel(const float* const* __restrict__ src, const int64_t* const* __restrict__ ts, size_t L,
                            size_t n, float* dst_p, float* dst_m, float* dst_v, int64_t* dst_t, float inv) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float sp = 0.0f, sm = 0.0f, sv = 0.0f;
    for (size_t a = 0; a < L; ++a) {
      sp += src[a][i];
      sm += src[L + a][i];
      sv += src[2 * L + a][i];
    }
    dst_p[i] = sp * inv;
    dst_m[i] = sm * inv;
    dst_v[i] = sv * inv;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // every counter read before the (possibly aliased) write
    int64_t t = 0;
    for (size_t a = 0; a < L; ++a) t = max(t, *ts[a]);
    *dst_t = t;
  }
}

// Rank candidates by (score desc, seq asc); a candidate's rank is the number
// of candidates that beat it.  Equals sequential leaderboard_update insertion
// (tournament.hpp:104-119; test_tournament.cpp:95-126).
__global__ void leaderboard_rank_kernel(const double* __restrict__ score, const uint64_t* __restrict__ seq, int n,
                                        int capacity, int32_t* __restrict__ order, int32_t* __restrict__ count,
                                        int32_t* __restrict__ status) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!isfinite(score[i])) bad = 1;
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) {
      status[0] = PRB_ERR_NUMERIC;
      *count = 0;
    }
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double si = score[i];
    const uint64_t qi = seq[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double sj = score[j];
      // (score desc, seq asc); duplicate (score, seq) keys fall back to the candidate index so
      // every rank is taken exactly once
      rank += (sj > si) || (sj == si && (seq[j] < qi || (seq[j] == qi && j < i)));
    }
    if (rank < capacity) order[rank] = i;
  }
  if (threadIdx.x == 0) {
    *count = min(n, capacity);
    status[0] = 0;
  }
}

// Leaderboard::refresh_stats (tournament.hpp:66-87): per-coordinate mean and population variance
// of the entries' flat parameters, in the reference's order -- sum over the entries in board
// order, times 1/n, then the sum of squared deviations times 1/n -- in fp64 with explicit
// round-to-nearest (the -ffp-contract=off reference build).  One thread per coordinate; every
// entry's params are read twice (n x 4 B x 2, L2 serves the second pass for a board of <= 10).
__global__ void population_stats_kernel(const float* const* __restrict__ entries, int n, size_t P,
                                        double* __restrict__ mean, double* __restrict__ var) {
  const double inv = 1.0 / (double)n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (size_t)gridDim.x * blockDim.x) {
    double m = 0.0;
    for (int e = 0; e < n; ++e) m = __dadd_rn(m, (double)entries[e][i]);
    m = __dmul_rn(m, inv);
    double v = 0.0;
    for (int e = 0; e < n; ++e) {
      const double d = __dsub_rn((double)entries[e][i], m);
      v = __dadd_rn(v, __dmul_rn(d, d));
    }
    mean[i] = m;
    var[i] = __dmul_rn(v, inv);
  }
}

// artifact_init (artifact.hpp:91-105) on the device: policy_init's actor MLP from
// mt19937_64(derive_seed(seed, kInit, 1)) and the critic from mt19937_64(derive_seed(seed, kInit,
// 2)), each layer's weights drawn row-major from uniform_real_distribution(-1/sqrt(fan_in),
// +1/sqrt(fan_in)) (nn.hpp:40-54) -- the reference's own generator and draw order, so the fp32
// parameters are the reference's values rounded once.  Thread 0 draws the actor, thread 1 the
// critic (two independent streams); biases and log_std are zero (the caller's memset).
struct InitNet {
  int nl;
  int dims[kMaxLayers + 1];
  int off[kMaxLayers];
  uint64_t seed;
};

// mlp_init (nn.hpp:40-54) for both nets, CTA k = net k, the reference's mt19937_64 stream
// (derive_seed(seed, kInit, k + 1)) generated 312 words at a time in parallel: the twist of a
// block is three data-parallel phases (words [0,156) read only old words; [156,311) read the
// new words 156 below them; word 311 reads new words 0 and 155 -- the serial loop's
// dependencies exactly), then thread i tempers word i and turns draw 312 b + i into its weight
// (uniform_real_distribution(-1/sqrt(fan_in), +) over generate_canonical<double, 53>: one
// 64-bit draw per weight).  Bit-identical to the serial stream; ~40x faster than one thread
// per net, which a generation's fresh pods used to wait ~2.3 ms for.
__global__ void __launch_bounds__(320) artifact_init_kernel(float* __restrict__ params, InitNet actor, InitNet critic) {
  __shared__ uint64_t mt[kMtN];
  const InitNet& n = blockIdx.x == 0 ? actor : critic;
  const int t = threadIdx.x;
  if (t == 0) mt64_seed(mt, 1, n.seed);
  int total = 0;
  for (int l = 0; l < n.nl; ++l) total += n.dims[l] * n.dims[l + 1];
  __syncthreads();
  constexpr uint64_t kUp = 0xFFFFFFFF80000000ULL, kLo = 0x7FFFFFFFULL, kMag = 0xB5026F5AA96619E9ULL;
  auto twist_word = [&](uint64_t cur, uint64_t nxt, uint64_t far) {
    const uint64_t y = (cur & kUp) | (nxt & kLo);
    return far ^ (y >> 1) ^ ((y & 1ULL) ? kMag : 0ULL);
  };
  for (int k0 = 0; k0 < total; k0 += kMtN) {
    uint64_t v = 0;
    if (t < 156) v = twist_word(mt[t], mt[t + 1], mt[t + 156]);
    __syncthreads();
    if (t < 156) mt[t] = v;
    __syncthreads();
    if (t >= 156 && t < kMtN - 1) v = twist_word(mt[t], mt[t + 1], mt[t - 156]);
    __syncthreads();
    if (t >= 156 && t < kMtN - 1) mt[t] = v;
    if (t == 0) mt[kMtN - 1] = twist_word(mt[kMtN - 1], mt[0], mt[155]);
    __syncthreads();
    const int k = k0 + t;
    if (t < kMtN && k < total) {
      uint64_t x = mt[t];
      x ^= (x >> 29) & 0x5555555555555555ULL;
      x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
      x ^= (x << 37) & 0xFFF7EEE000000000ULL;
      x ^= (x >> 43);
      int l = 0, start = 0;
      while (k - start >= n.dims[l] * n.dims[l + 1]) {
        start += n.dims[l] * n.dims[l + 1];
        ++l;
      }
      const double scale = __ddiv_rn(1.0, __dsqrt_rn((double)n.dims[l]));
      double u = __dmul_rn(__ull2double_rn(x), 5.421010862427522170037264e-20);  // 2^-64
      if (u >= 1.0) u = 0.99999999999999988898;  // nextafter(1, 0)
      params[n.off[l] + (k - start)] = (float)__dadd_rn(__dmul_rn(u, __dsub_rn(scale, -scale)), -scale);
    }
    __syncthreads();  // the next twist overwrites the words just tempered
  }
}

__global__ void mutate_kernel(float* __restrict__ p, size_t n, uint64_t seed, float sigma) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const Philox4 r = philox4x32_10((uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)i, (uint32_t)(i >> 32),
                                    0x6d757461u /*"muta"*/, 0u);
    const float2 z = box_muller(r.x, r.y);
    p[i] += sigma * z.x;
  }
}

}  // namespace

void prb_agent_finite_gate_and_adam(prb_agent a, const float* d_grads, cudaStream_t s) {
  const int cgrid = (int)std::min<size_t>((a->P + 255) / 256, (size_t)a->ctx->num_sms * 8);
  finite_check_kernel<<<cgrid, 256, 0, s>>>(d_grads, a->P, a->d_status.p, a->d_t.p);
  const int grid = (int)std::min<size_t>((a->P + 255) / 256, (size_t)a->ctx->num_sms * 8);
  ProfScope prof(a->ctx, kProfAdam);
  adam_kernel<<<grid, 256, 0, s>>>(a->d_params.p, d_grads, a->d_m.p, a->d_v.p, a->P, a->d_t.p, a->d_status.p,
                                   (float)a->lr, a->beta1, a->beta2, (float)a->eps);
  PRB_CHECK_LAUNCH();
}

void prb_adam_launch(prb_agent a, const float* d_grads, const int32_t* gate, cudaStream_t s) {
  const int grid = (int)std::min<size_t>((a->P + 255) / 256, 1184);
  adam_kernel<<<grid, 256, 0, s>>>(a->d_params.p, d_grads, a->d_m.p, a->d_v.p, a->P, a->d_t.p, gate, (float)a->lr,
                                   a->beta1, a->beta2, (float)a->eps);
  PRB_CHECK_LAUNCH();
}

int prb_agent_status(prb_agent a, std::string* msg);

extern "C" {

int prb_agent_create(prb_ctx ctx, size_t S, size_t A, const size_t* hidden, int nh, prb_agent* out) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && out, PRB_ERR_USAGE, "prb_agent_create: NULL argument");
    PRB_REQUIRE(S > 0 && A > 0, PRB_ERR_USAGE, "mlp_init: need at least input and output dims");
    PRB_REQUIRE(nh >= 0 && nh <= 6, PRB_ERR_CONFIG, "prb_agent_create: 0..6 hidden layers supported");
    for (int i = 0; i < nh; ++i)
      PRB_REQUIRE(hidden[i] > 0 && hidden[i] <= 1024, PRB_ERR_CONFIG, "prb_agent_create: hidden widths 1..1024");
    PRB_REQUIRE(S <= 4096 && A <= 256, PRB_ERR_CONFIG, "prb_agent_create: state_dim <= 4096, action_dim <= 256");
    PRB_CUDA(cudaSetDevice(ctx->device));
    auto* a = new prb_agent_s;
    a->ctx = ctx;
    a->S = S;
    a->A = A;
    a->hidden.assign(hidden, hidden + nh);
    layout(a);
    // rounded up to whole 16-byte blocks (zero padding): the tensor-core PPO update bulk-copies
    // parameter slices whose ends are 16-byte aligned
    const size_t Palloc = (a->P + 3) & ~size_t(3);
    a->d_params.alloc(Palloc);
    a->d_m.alloc(Palloc);
    a->d_v.alloc(Palloc);
    a->d_grads.alloc(Palloc);
    a->d_t.alloc(1);
    a->d_status.alloc(4);
    // on the agent's (non-blocking) stream, then waited: a legacy-stream cudaMemset would not be
    // ordered with work the caller enqueues on any context stream afterwards
    cudaStream_t s = a->ctx->stream;
    PRB_CUDA(cudaMemsetAsync(a->d_params.p, 0, a->d_params.bytes(), s));
    PRB_CUDA(cudaMemsetAsync(a->d_m.p, 0, a->d_m.bytes(), s));
    PRB_CUDA(cudaMemsetAsync(a->d_v.p, 0, a->d_v.bytes(), s));
    PRB_CUDA(cudaMemsetAsync(a->d_t.p, 0, sizeof(int64_t), s));
    PRB_CUDA(cudaMemsetAsync(a->d_status.p, 0, 4 * sizeof(int32_t), s));
    PRB_CUDA(cudaStreamSynchronize(s));
    *out = a;
  });
}

int prb_agent_destroy(prb_agent a) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    if (a) cudaStreamSynchronize(a->ctx->stream);
    delete a;
  });
}

size_t prb_agent_param_count(prb_agent a) { return a ? a->P : 0; }
float* prb_agent_params_device(prb_agent a) { return a ? a->d_params.p : nullptr; }

int prb_agent_set_host(prb_agent a, const double* flat, const double* m, const double* v, int64_t t, double lr) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && flat, PRB_ERR_USAGE, "prb_agent_set_host: NULL argument");
    std::vector<float> buf(a->P);
    cudaStream_t s = a->ctx->stream;
    for (size_t i = 0; i < a->P; ++i) buf[i] = (float)flat[i];
    PRB_CUDA(cudaMemcpyAsync(a->d_params.p, buf.data(), a->P * sizeof(float), cudaMemcpyHostToDevice, s));
    a->ctx->sync();
    if (m) {
      for (size_t i = 0; i < a->P; ++i) buf[i] = (float)m[i];
      PRB_CUDA(cudaMemcpyAsync(a->d_m.p, buf.data(), a->P * sizeof(float), cudaMemcpyHostToDevice, s));
      a->ctx->sync();
    } else {
      PRB_CUDA(cudaMemsetAsync(a->d_m.p, 0, a->d_m.bytes(), s));
    }
    if (v) {
      for (size_t i = 0; i < a->P; ++i) buf[i] = (float)v[i];
      PRB_CUDA(cudaMemcpyAsync(a->d_v.p, buf.data(), a->P * sizeof(float), cudaMemcpyHostToDevice, s));
      a->ctx->sync();
    } else {
      PRB_CUDA(cudaMemsetAsync(a->d_v.p, 0, a->d_v.bytes(), s));
    }
    PRB_CUDA(cudaMemcpyAsync(a->d_t.p, &t, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    a->ctx->sync();
    a->lr = lr;
  });
}

int prb_agent_get_host(prb_agent a, double* flat, double* m, double* v, int64_t* t) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a, PRB_ERR_USAGE, "prb_agent_get_host: NULL agent");
    std::vector<float> buf(a->P);
    cudaStream_t s = a->ctx->stream;
    auto pull = [&](const float* d, double* h) {
      if (!h) return;
      PRB_CUDA(cudaMemcpyAsync(buf.data(), d, a->P * sizeof(float), cudaMemcpyDeviceToHost, s));
      a->ctx->sync();
      for (size_t i = 0; i < a->P; ++i) h[i] = buf[i];
    };
    pull(a->d_params.p, flat);
    pull(a->d_m.p, m);
    pull(a->d_v.p, v);
    if (t) {
      PRB_CUDA(cudaMemcpyAsync(t, a->d_t.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      a->ctx->sync();
    }
  });
}

int prb_agent_copy(prb_agent dst, prb_agent src) {
  return guard([&] {
    DeviceScope dev_(dst ? dst->ctx : nullptr);
    PRB_REQUIRE(dst && src, PRB_ERR_USAGE, "prb_agent_copy: NULL agent");
    PRB_REQUIRE(dst->P == src->P && dst->adims == src->adims && dst->cdims == src->cdims, PRB_ERR_USAGE,
                "prb_agent_copy: incompatible shapes");
    cudaStream_t s = src->ctx->stream;
    PRB_CUDA(cudaMemcpyAsync(dst->d_params.p, src->d_params.p, src->d_params.bytes(), cudaMemcpyDeviceToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(dst->d_m.p, src->d_m.p, src->d_m.bytes(), cudaMemcpyDeviceToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(dst->d_v.p, src->d_v.p, src->d_v.bytes(), cudaMemcpyDeviceToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(dst->d_t.p, src->d_t.p, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (dst->ctx->stream != s) src->ctx->sync();
    dst->lr = src->lr;
  });
}

int prb_adam_step_host(prb_agent a, const double* grads) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && grads, PRB_ERR_USAGE, "prb_adam_step_host: NULL argument");
    for (size_t i = 0; i < a->P; ++i)  // nn.hpp:169-171: reject before touching state
      PRB_REQUIRE(std::isfinite(grads[i]), PRB_ERR_NUMERIC, "adam_step: non-finite gradient, step aborted");
    std::vector<float> g(a->P);
    for (size_t i = 0; i < a->P; ++i) g[i] = (float)grads[i];
    cudaStream_t s = a->ctx->stream;
    PRB_CUDA(cudaMemcpyAsync(a->d_grads.p, g.data(), a->P * sizeof(float), cudaMemcpyHostToDevice, s));
    prb_agent_finite_gate_and_adam(a, a->d_grads.p, s);
    a->ctx->sync();
  });
}

int prb_adam_step_device(prb_agent a, const float* d_grads) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && d_grads, PRB_ERR_USAGE, "prb_adam_step_device: NULL argument");
    cudaStream_t s = a->ctx->stream;
    prb_agent_finite_gate_and_adam(a, d_grads, s);
    int32_t st[2];
    PRB_CUDA(cudaMemcpyAsync(st, a->d_status.p, sizeof(st), cudaMemcpyDeviceToHost, s));
    a->ctx->sync();
    if (st[0] != 0) {
      PRB_CUDA(cudaMemsetAsync(a->d_status.p, 0, 2 * sizeof(int32_t), s));
      a->ctx->sync();
      fail(st[0], "adam_step: non-finite gradient, step aborted");
    }
  });
}

int prb_fuse_parameters(const prb_agent* agents, size_t n, prb_agent out) {
  return guard([&] {
    DeviceScope dev_(out ? out->ctx : nullptr);
    PRB_REQUIRE(n > 0 && agents, PRB_ERR_USAGE, "fuse_parameters: empty artifact list");  // pod.hpp:142
    PRB_REQUIRE(out, PRB_ERR_USAGE, "fuse_parameters: NULL output");
    for (size_t i = 0; i < n; ++i)
      PRB_REQUIRE(agents[i] && agents[i]->adims == agents[0]->adims && agents[i]->cdims == agents[0]->cdims &&
                      agents[i]->A == agents[0]->A,
                  PRB_ERR_USAGE, "fuse_parameters: artifacts have incompatible shapes");  // pod.hpp:145-148
    PRB_REQUIRE(out->P == agents[0]->P, PRB_ERR_USAGE, "fuse_parameters: output shape mismatch");
    prb_ctx_s* ctx = out->ctx;
    cudaStream_t s = ctx->stream;
    for (size_t i = 0; i < n; ++i)
      if (agents[i]->ctx->stream != s) agents[i]->ctx->sync();
    if (n == 1) {  // a single artifact is returned unchanged (pod.hpp:143)
      if (agents[0] != out) {
        int rc = prb_agent_copy(out, agents[0]);
        if (rc) fail(rc, prb_last_error());
      }
      return;
    }
    // mean of params, m, v; t = max (pod.hpp:149-171) -- one kernel, no host round trips
    std::vector<const void*> all(4 * n);
    for (size_t i = 0; i < n; ++i) {
      all[i] = agents[i]->d_params.p;
      all[n + i] = agents[i]->d_m.p;
      all[2 * n + i] = agents[i]->d_v.p;
      all[3 * n + i] = agents[i]->d_t.p;
    }
    const void** dptr = static_cast<const void**>(ctx->device_scratch(4 * n * sizeof(void*)));
    PRB_CUDA(cudaMemcpyAsync(dptr, all.data(), all.size() * sizeof(void*), cudaMemcpyHostToDevice, s));
    const float inv = (float)(1.0 / (double)n);
    const size_t P = out->P;
    const int grid = (int)std::min<size_t>((P + 255) / 256, 1184);
    fuse_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const float* const*>(dptr),
                                     reinterpret_cast<const int64_t* const*>(dptr + 3 * n), n, P, out->d_params.p,
                                     out->d_m.p, out->d_v.p, out->d_t.p, inv);
    PRB_CHECK_LAUNCH();
    out->lr = agents[0]->lr;
    ctx->sync();
  });
}

int prb_leaderboard_rank(prb_ctx ctx, const double* d_scores, const uint64_t* d_seqs, size_t n, size_t capacity,
                         int32_t* d_order, int32_t* d_count) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx, PRB_ERR_USAGE, "prb_leaderboard_rank: NULL ctx");
    PRB_REQUIRE(capacity > 0, PRB_ERR_CONFIG, "Leaderboard: capacity must be > 0");  // tournament.hpp:47
    PRB_REQUIRE(n < (1u << 20), PRB_ERR_CONFIG, "prb_leaderboard_rank: too many candidates");
    int32_t* status = static_cast<int32_t*>(ctx->device_scratch(16));
    leaderboard_rank_kernel<<<1, 256, 0, ctx->stream>>>(d_scores, d_seqs, (int)n, (int)capacity, d_order, d_count,
                                                        status);
    PRB_CHECK_LAUNCH();
    int32_t st = 0;
    PRB_CUDA(cudaMemcpyAsync(&st, status, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    PRB_REQUIRE(st == 0, PRB_ERR_NUMERIC, "leaderboard_update: candidate score is not finite");
  });
}

int prb_leaderboard_rank_host(prb_ctx ctx, const double* scores, const uint64_t* seqs, size_t n, size_t capacity,
                              int32_t* order, int32_t* count) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx, PRB_ERR_USAGE, "prb_leaderboard_rank_host: NULL ctx");
    DevBuf<double> ds;
    DevBuf<uint64_t> dq;
    DevBuf<int32_t> dout;
    ds.alloc(std::max<size_t>(n, 1));
    dq.alloc(std::max<size_t>(n, 1));
    dout.alloc(capacity + 1);
    cudaStream_t s = ctx->stream;
    if (n) {
      PRB_CUDA(cudaMemcpyAsync(ds.p, scores, n * sizeof(double), cudaMemcpyHostToDevice, s));
      PRB_CUDA(cudaMemcpyAsync(dq.p, seqs, n * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    }
    int rc = prb_leaderboard_rank(ctx, ds.p, dq.p, n, capacity, dout.p, dout.p + capacity);
    if (rc) fail(rc, prb_last_error());
    std::vector<int32_t> h(capacity + 1);
    PRB_CUDA(cudaMemcpyAsync(h.data(), dout.p, (capacity + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    ctx->sync();
    *count = h[capacity];
    for (int i = 0; i < *count; ++i) order[i] = h[i];
  });
}

int prb_agent_init_device(prb_agent a, uint64_t seed, double lr) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a, PRB_ERR_USAGE, "prb_agent_init_device: NULL agent");
    cudaStream_t s = a->ctx->stream;
    PRB_CUDA(cudaMemsetAsync(a->d_params.p, 0, a->d_params.bytes(), s));  // biases, log_std (0)
    PRB_CUDA(cudaMemsetAsync(a->d_m.p, 0, a->d_m.bytes(), s));            // adam_init (nn.hpp:155-160)
    PRB_CUDA(cudaMemsetAsync(a->d_v.p, 0, a->d_v.bytes(), s));
    PRB_CUDA(cudaMemsetAsync(a->d_t.p, 0, sizeof(int64_t), s));
    InitNet nets[2];
    for (int k = 0; k < 2; ++k) {
      const std::vector<size_t>& d = k == 0 ? a->adims : a->cdims;
      const std::vector<size_t>& off = k == 0 ? a->aoff : a->coff;
      PRB_REQUIRE(d.size() <= (size_t)kMaxLayers + 1, PRB_ERR_CONFIG, "prb_agent_init_device: too many layers");
      nets[k].nl = (int)d.size() - 1;
      for (size_t i = 0; i < d.size(); ++i) nets[k].dims[i] = (int)d[i];
      for (size_t i = 0; i < off.size(); ++i) nets[k].off[i] = (int)off[i];
      nets[k].seed = derive_seed(seed, {5 /*kInit*/, (uint64_t)(k + 1)});
    }
    artifact_init_kernel<<<2, 320, 0, s>>>(a->d_params.p, nets[0], nets[1]);
    PRB_CHECK_LAUNCH();
    a->lr = lr;
    a->ctx->sync();
  });
}

int prb_leaderboard_stats(const prb_agent* entries, size_t n, double* d_mean, double* d_variance) {
  return guard([&] {
    PRB_REQUIRE(entries && d_mean && d_variance, PRB_ERR_USAGE, "prb_leaderboard_stats: NULL argument");
    if (n == 0) return;  // an empty board has empty stats (tournament.hpp:69)
    for (size_t i = 0; i < n; ++i)
      PRB_REQUIRE(entries[i] && entries[i]->P == entries[0]->P && entries[i]->ctx->device == entries[0]->ctx->device,
                  PRB_ERR_USAGE, "prb_leaderboard_stats: entries have different shapes or devices");
    PRB_REQUIRE(n < (1u << 20), PRB_ERR_CONFIG, "prb_leaderboard_stats: too many entries");
    prb_ctx_s* ctx = entries[0]->ctx;
    DeviceScope dev(ctx);
    cudaStream_t s = ctx->stream;
    for (size_t i = 1; i < n; ++i)
      if (entries[i]->ctx->stream != s) entries[i]->ctx->sync();
    std::vector<const float*> hp(n);
    for (size_t i = 0; i < n; ++i) hp[i] = entries[i]->d_params.p;
    DevBuf<const float*> dp;
    dp.alloc(n);
    PRB_CUDA(cudaMemcpyAsync(dp.p, hp.data(), n * sizeof(float*), cudaMemcpyHostToDevice, s));
    const size_t P = entries[0]->P;
    const int grid = (int)std::min<size_t>((P + 255) / 256, (size_t)ctx->num_sms * 8);
    population_stats_kernel<<<grid, 256, 0, s>>>(dp.p, (int)n, P, d_mean, d_variance);
    PRB_CHECK_LAUNCH();
    ctx->sync();  // dp is released on return
  });
}

int prb_leaderboard_stats_host(const prb_agent* entries, size_t n, double* mean, double* variance) {
  return guard([&] {
    PRB_REQUIRE(entries && mean && variance, PRB_ERR_USAGE, "prb_leaderboard_stats_host: NULL argument");
    if (n == 0) return;
    PRB_REQUIRE(entries[0], PRB_ERR_USAGE, "prb_leaderboard_stats_host: NULL entry");
    DeviceScope dev(entries[0]->ctx);
    const size_t P = entries[0]->P;
    DevBuf<double> d;
    d.alloc(2 * P);
    int rc = prb_leaderboard_stats(entries, n, d.p, d.p + P);
    if (rc) fail(rc, prb_last_error());
    PRB_CUDA(cudaMemcpy(mean, d.p, P * sizeof(double), cudaMemcpyDeviceToHost));
    PRB_CUDA(cudaMemcpy(variance, d.p + P, P * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int prb_debug_agent_grads(prb_agent a, double* grads) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && grads, PRB_ERR_USAGE, "prb_debug_agent_grads: NULL argument");
    std::vector<float> g(a->P);
    PRB_CUDA(cudaMemcpyAsync(g.data(), a->d_grads.p, a->P * sizeof(float), cudaMemcpyDeviceToHost, a->ctx->stream));
    a->ctx->sync();
    for (size_t i = 0; i < a->P; ++i) grads[i] = g[i];
  });
}

int prb_agent_set_ppo_mode(prb_agent a, int mode) {
  return guard([&] {
    PRB_REQUIRE(a, PRB_ERR_USAGE, "prb_agent_set_ppo_mode: NULL agent");
    PRB_REQUIRE(mode == 0 || mode == 1, PRB_ERR_CONFIG, "prb_agent_set_ppo_mode: mode must be 0 or 1");
    a->ppo_mode = mode;
  });
}

int prb_agent_mutate(prb_agent a, uint64_t mutation_seed, double sigma) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a, PRB_ERR_USAGE, "prb_agent_mutate: NULL agent");
    cudaStream_t s = a->ctx->stream;
    if (sigma > 0.0) {
      const int grid = (int)std::min<size_t>((a->P + 255) / 256, 1184);
      mutate_kernel<<<grid, 256, 0, s>>>(a->d_params.p, a->P, mutation_seed, (float)sigma);
      PRB_CHECK_LAUNCH();
    }
    PRB_CUDA(cudaMemsetAsync(a->d_t.p, 0, sizeof(int64_t), s));  // optimizer.t = 0 (tournament.hpp:160)
    a->ctx->sync();
  });
}

}  // extern "C"
