// api_core.cu -- context, memory, errors, seeds, market data and artifact
// initialisation for the prb_* C ABI.  Host code; the market feature table
// and price table it builds are the device-resident inputs of the env kernels.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>

#include "prb_internal.h"
#include "rng.cuh"
#include "tmap.h"

namespace prb {

static thread_local std::string g_last_error;
static thread_local int g_last_code = 0;

void set_last_error(int code, const std::string& msg) {
  g_last_code = code;
  g_last_error = msg;
}

void ensure_smem_attr(const void* kernel, size_t smem_bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, size_t>> done;  // ((kernel, device), bytes)
  int dev = 0;
  PRB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done)
    if (e.first.first == kernel && e.first.second == dev && e.second >= smem_bytes) return;
  PRB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
  done.push_back({{kernel, dev}, smem_bytes});
}

static std::atomic<int> g_options[8];

int debug_option(int option) { return (option > 0 && option < 8) ? g_options[option].load() : 0; }

const char* debug_env(const char* name) {
#ifdef PRB_DEBUG_KNOBS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

void encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, uint64_t dim0, uint64_t dim1,
                    uint64_t stride1_bytes, uint32_t box0, uint32_t box1, CUtensorMapL2promotion l2) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static const Fn fn = [] {  // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PRB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    PRB_REQUIRE(p && q == cudaDriverEntryPointSuccess, PRB_ERR_CUDA, "cuTensorMapEncodeTiled not available");
    return reinterpret_cast<Fn>(p);
  }();
  const cuuint64_t dims[2] = {dim0, dim1};
  const cuuint64_t strides[1] = {stride1_bytes};
  const cuuint32_t box[2] = {box0, box1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  PRB_REQUIRE(r == CUDA_SUCCESS, PRB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

uint64_t splitmix64(uint64_t x) { return splitmix64_d(x); }

uint64_t derive_seed(uint64_t base, std::initializer_list<uint64_t> tags) {
  uint64_t s = splitmix64(base);
  for (uint64_t t : tags) s = splitmix64(s ^ splitmix64(t));
  return s;
}

}  // namespace prb

using namespace prb;

void* prb_ctx_s::pinned_staging(size_t bytes) {
  if (bytes > pinned_bytes) {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    PRB_CUDA(cudaMallocHost(&pinned, bytes));
    pinned_bytes = bytes;
  }
  return pinned;
}

void* prb_ctx_s::device_scratch(size_t bytes) {
  if (bytes > scratch_bytes) {
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    PRB_CUDA(cudaMalloc(&scratch, bytes));
    scratch_bytes = bytes;
  }
  return scratch;
}

unsigned int* prb_ctx_s::last_cta_counter() {
  if (!done_counter) {
    PRB_CUDA(cudaMalloc(&done_counter, sizeof(unsigned int)));
    PRB_CUDA(cudaMemsetAsync(done_counter, 0, sizeof(unsigned int), stream));
  }
  return done_counter;
}

void prb_ctx_s::sync() { PRB_CUDA(cudaStreamSynchronize(stream)); }

cudaEvent_t prb_ctx_s::take_event() {
  if (ev_pool.empty()) {
    cudaEvent_t e;
    PRB_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = ev_pool.back();
  ev_pool.pop_back();
  return e;
}

extern "C" {

const char* prb_last_error(void) { return g_last_error.c_str(); }
int prb_version(void) { return 1; }

int prb_debug_set_option(int option, int value) {
  return guard([&] {
    PRB_REQUIRE(option > 0 && option < 8, PRB_ERR_USAGE, "prb_debug_set_option: unknown option");
    g_options[option].store(value);
  });
}

uint64_t prb_splitmix64(uint64_t x) { return splitmix64(x); }

uint64_t prb_derive_seed(uint64_t base, const uint64_t* tags, int n) {
  uint64_t s = splitmix64(base);
  for (int i = 0; i < n; ++i) s = splitmix64(s ^ splitmix64(tags[i]));
  return s;
}

int prb_ctx_create(int device, prb_ctx* out) {
  return guard([&] {
    PRB_REQUIRE(out, PRB_ERR_USAGE, "prb_ctx_create: out is NULL");
    int n = 0;
    PRB_CUDA(cudaGetDeviceCount(&n));
    PRB_REQUIRE(device >= 0 && device < n, PRB_ERR_CONFIG, "prb_ctx_create: no CUDA device " + std::to_string(device));
    PRB_CUDA(cudaSetDevice(device));
    auto* c = new prb_ctx_s;
    c->device = device;
    PRB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    PRB_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    *out = c;
  });
}

int prb_ctx_destroy(prb_ctx c) {
  return guard([&] {
    DeviceScope dev_(c);
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->scratch) cudaFree(c->scratch);
    if (c->done_counter) cudaFree(c->done_counter);
    cudaStreamDestroy(c->stream);
    delete c;
  });
}

int prb_ctx_synchronize(prb_ctx c) { return guard([&] { c->sync(); }); }

int prb_ctx_profile(prb_ctx c, int enable) {
  return guard([&] {
    DeviceScope dev_(c);
    PRB_REQUIRE(c, PRB_ERR_USAGE, "prb_ctx_profile: NULL ctx");
    c->sync();
    for (auto& e : c->ev_live) {
      c->ev_pool.push_back(e.a);
      c->ev_pool.push_back(e.b);
    }
    c->ev_live.clear();
    for (int i = 0; i < 16; ++i) {
      c->prof_ms[i] = 0.0;
      c->prof_n[i] = 0;
    }
    c->profiling = enable != 0;
  });
}

int prb_ctx_profile_read(prb_ctx c, int kind, double* total_ms, uint64_t* launches) {
  return guard([&] {
    DeviceScope dev_(c);
    PRB_REQUIRE(c && kind >= 0 && kind < 16, PRB_ERR_USAGE, "prb_ctx_profile_read: bad argument");
    c->sync();
    for (auto& e : c->ev_live) {
      float ms = 0.f;
      PRB_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
      c->prof_ms[e.kind] += ms;
      c->prof_n[e.kind] += 1;
      c->ev_pool.push_back(e.a);
      c->ev_pool.push_back(e.b);
    }
    c->ev_live.clear();
    if (total_ms) *total_ms = c->prof_ms[kind];
    if (launches) *launches = c->prof_n[kind];
  });
}
void* prb_ctx_stream(prb_ctx c) { return c ? (void*)c->stream : nullptr; }

int prb_device_alloc(prb_ctx c, size_t bytes, void** out) {
  return guard([&] {
    DeviceScope dev_(c);
    PRB_CUDA(cudaSetDevice(c->device));
    PRB_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  });
}
int prb_device_free(prb_ctx, void* p) { return guard([&] { PRB_CUDA(cudaFree(p)); }); }
int prb_memcpy_h2d(prb_ctx c, void* d, const void* s, size_t n) {
  return guard([&] {
    DeviceScope dev_(c);
    PRB_CUDA(cudaMemcpyAsync(d, s, n, cudaMemcpyHostToDevice, c->stream));
    c->sync();
  });
}
int prb_memcpy_d2h(prb_ctx c, void* d, const void* s, size_t n) {
  return guard([&] {
    DeviceScope dev_(c);
    PRB_CUDA(cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  });
}
int prb_memcpy_h2d_async(prb_ctx c, void* d, const void* s, size_t n) {
  return guard([&] { PRB_CUDA(cudaMemcpyAsync(d, s, n, cudaMemcpyHostToDevice, c->stream)); });
}
int prb_memcpy_d2h_async(prb_ctx c, void* d, const void* s, size_t n) {
  return guard([&] { PRB_CUDA(cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToHost, c->stream)); });
}

// ---------------------------------------------------------------------------
// Market data.
// ---------------------------------------------------------------------------

int prb_market_synthetic(uint64_t seed, int K, size_t T, double* open, double* high, double* low, double* close,
                         double* volume) {
  return guard([&] {
    PRB_REQUIRE(K > 0 && T > 0, PRB_ERR_CONFIG, "prb_market_synthetic: K and T must be > 0");
    // mt19937_64(seed); p0_k ~ U(10,200) for k = 0..K-1, then
    // for t = 1..T-1, k = 0..K-1: p_k[t] = p_k[t-1] * exp(1e-3 * N(0,1)).
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u0(10.0, 200.0);
    std::normal_distribution<double> nrm(0.0, 1.0);
    std::vector<double> p((size_t)K * T);
    for (int k = 0; k < K; ++k) p[(size_t)k * T] = u0(rng);
    for (size_t t = 1; t < T; ++t)
      for (int k = 0; k < K; ++k) p[(size_t)k * T + t] = p[(size_t)k * T + t - 1] * std::exp(1e-3 * nrm(rng));
    for (size_t i = 0; i < p.size(); ++i) {
      if (close) close[i] = p[i];
      if (open) open[i] = p[i];
      if (high) high[i] = 1.001 * p[i];
      if (low) low[i] = 0.999 * p[i];
      if (volume) volume[i] = 1000.0;
    }
  });
}

int prb_compute_indicators(const double* high, const double* low, const double* close, size_t T, int K,
                           double* out) {
  return guard([&] {
    // market.hpp:373-392; ordering macd, rsi_14, cci_30, sma_20 (:101)
    PRB_REQUIRE(T >= 35, PRB_ERR_DATA,
                "compute_indicators: need at least 35 rows, have " + std::to_string(T));
    std::vector<double> fast(T), slow(T), tp(T);
    auto ema = [&](const double* x, size_t period, std::vector<double>& o) {
      const double alpha = 2.0 / (static_cast<double>(period) + 1.0);
      o[0] = x[0];
      for (size_t t = 1; t < T; ++t) o[t] = alpha * x[t] + (1.0 - alpha) * o[t - 1];
    };
    auto fill_head = [&](double* x, size_t first) {
      for (size_t t = 0; t < first && t < T; ++t) x[t] = x[first];
    };
    for (int k = 0; k < K; ++k) {
      const double* c = close + (size_t)k * T;
      const double* h = high + (size_t)k * T;
      const double* l = low + (size_t)k * T;
      double* macd = out + ((size_t)0 * K + k) * T;
      double* rsi = out + ((size_t)1 * K + k) * T;
      double* cci = out + ((size_t)2 * K + k) * T;
      double* sma = out + ((size_t)3 * K + k) * T;
      ema(c, 12, fast);
      ema(c, 26, slow);
      for (size_t t = 0; t < T; ++t) macd[t] = fast[t] - slow[t];
      // Wilder RSI(14)
      const size_t rp = 14;
      double gain = 0.0, loss = 0.0;
      for (size_t t = 1; t <= rp; ++t) {
        const double d = c[t] - c[t - 1];
        gain += std::max(d, 0.0);
        loss += std::max(-d, 0.0);
      }
      gain /= static_cast<double>(rp);
      loss /= static_cast<double>(rp);
      auto rsi_value = [](double g, double l) {
        if (g == 0.0 && l == 0.0) return 50.0;
        if (l == 0.0) return 100.0;
        return 100.0 - 100.0 / (1.0 + g / l);
      };
      for (size_t t = 0; t < T; ++t) rsi[t] = 50.0;
      rsi[rp] = rsi_value(gain, loss);
      for (size_t t = rp + 1; t < T; ++t) {
        const double d = c[t] - c[t - 1];
        gain = (gain * static_cast<double>(rp - 1) + std::max(d, 0.0)) / static_cast<double>(rp);
        loss = (loss * static_cast<double>(rp - 1) + std::max(-d, 0.0)) / static_cast<double>(rp);
        rsi[t] = rsi_value(gain, loss);
      }
      fill_head(rsi, rp);
      // CCI(30) on the typical price
      const size_t cp = 30;
      for (size_t t = 0; t < T; ++t) tp[t] = (h[t] + l[t] + c[t]) / 3.0;
      for (size_t t = 0; t < T; ++t) cci[t] = 0.0;
      for (size_t t = cp - 1; t < T; ++t) {
        double mean = 0.0;
        for (size_t q = t + 1 - cp; q <= t; ++q) mean += tp[q];
        mean /= static_cast<double>(cp);
        double mad = 0.0;
        for (size_t q = t + 1 - cp; q <= t; ++q) mad += std::abs(tp[q] - mean);
        mad /= static_cast<double>(cp);
        cci[t] = (mad == 0.0) ? 0.0 : (tp[t] - mean) / (0.015 * mad);
      }
      fill_head(cci, cp - 1);
      // SMA(20)
      const size_t sp = 20;
      double win = 0.0;
      for (size_t t = 0; t < T; ++t) {
        sma[t] = 0.0;
        win += c[t];
        if (t >= sp) win -= c[t - sp];
        if (t + 1 >= sp) sma[t] = win / static_cast<double>(sp);
      }
      fill_head(sma, sp - 1);
    }
    for (size_t i = 0; i < (size_t)4 * K * T; ++i)
      PRB_REQUIRE(std::isfinite(out[i]), PRB_ERR_NUMERIC, "compute_indicators: non-finite indicator value");
  });
}

int prb_market_create(prb_ctx ctx, const double* close, const double* indicators, size_t T, int K, prb_market* out) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && out && close, PRB_ERR_USAGE, "prb_market_create: NULL argument");
    PRB_REQUIRE(K > 0 && T >= 2, PRB_ERR_DIMENSION, "prb_market_create: need K > 0 tickers and T >= 2 rows");
    PRB_CUDA(cudaSetDevice(ctx->device));
    auto* m = new prb_market_s;
    m->ctx = ctx;
    m->K = K;
    m->T = T;
    m->close.assign(close, close + (size_t)K * T);
    if (indicators) m->indicators.assign(indicators, indicators + (size_t)4 * K * T);
    std::vector<double> tk((size_t)T * K);
    for (int k = 0; k < K; ++k)
      for (size_t t = 0; t < T; ++t) tk[t * K + k] = close[(size_t)k * T + t];
    m->d_close_tk.alloc(tk.size());
    PRB_CUDA(cudaMemcpyAsync(m->d_close_tk.p, tk.data(), tk.size() * sizeof(double), cudaMemcpyHostToDevice,
                             m->ctx->stream));
    PRB_CUDA(cudaStreamSynchronize(m->ctx->stream));  // creation-time: visible to every stream
    *out = m;
  });
}

int prb_market_destroy(prb_market m) {
  return guard([&] { delete m; });
}

// ---------------------------------------------------------------------------
// artifact_init artifact.hpp:91-105 (policy_init nn.hpp:190-205, mlp_init
// nn.hpp:40-54): host-side, same mt19937_64 + uniform_real_distribution draws.
// ---------------------------------------------------------------------------

static void mlp_init_into(const std::vector<size_t>& dims, uint64_t seed, std::vector<double>& out) {
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i + 1 < dims.size(); ++i) {
    const double scale = 1.0 / std::sqrt(static_cast<double>(dims[i]));
    std::uniform_real_distribution<double> dist(-scale, scale);
    for (size_t j = 0; j < dims[i] * dims[i + 1]; ++j) out.push_back(dist(rng));
    for (size_t j = 0; j < dims[i + 1]; ++j) out.push_back(0.0);
  }
}

int prb_artifact_init(size_t S, size_t A, uint64_t seed, const size_t* hidden, int nh, double* flat_out,
                      size_t* param_count) {
  return guard([&] {
    PRB_REQUIRE(S > 0 && A > 0, PRB_ERR_USAGE, "artifact_init: state/action dims must be > 0");
    std::vector<size_t> ad{S}, cd{S};
    for (int i = 0; i < nh; ++i) {
      ad.push_back(hidden[i]);
      cd.push_back(hidden[i]);
    }
    ad.push_back(A);
    cd.push_back(1);
    std::vector<double> flat;
    mlp_init_into(ad, derive_seed(seed, {5 /*kInit*/, 1}), flat);
    for (size_t d = 0; d < A; ++d) flat.push_back(0.0);  // initial_log_std = 0
    mlp_init_into(cd, derive_seed(seed, {5, 2}), flat);
    if (param_count) *param_count = flat.size();
    if (flat_out) std::memcpy(flat_out, flat.data(), flat.size() * sizeof(double));
  });
}

}  // extern "C"
