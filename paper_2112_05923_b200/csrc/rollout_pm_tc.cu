// rollout_pm_tc.cu -- worker_collect (pod.hpp:95-132) for the PointMass2D
// VecEnv (env.hpp:84-146) with the configs[2] 3x256 actor/critic
// (6-256-256-256-2 / 6-256-256-256-1, tanh) on the 5th-gen tensor cores.
//
// The 3x256 weights (557 KB as bf16) do not fit one SM, so they are STREAMED:
// a one-off pack kernel lays them out in HBM as bf16 chunks ([256 N][32 K],
// 16 KB) already in the UMMA K-major operand layout, and producer warps stream
// them (L2-resident after the first tile) through a 5-slot shared-memory ring
// with 1-D bulk async copies (TMA engine, mbarrier transaction counts), in the
// exact order the single MMA issuer consumes them.  One persistent CTA per SM,
// 384 threads.  The actor and the critic are two chains that share only the obs
// tile; the critic runs one epilogue behind the actor so that one net's
// epilogue overlaps the other net's MMAs:
//   warps 0-3   actor epilogues (TMEM -> +b, tanh -> bf16 operand), obs tile,
//               Philox sample + log-prob, PointMass step in fp64, rollout rows
//   warps 4-7   critic epilogues, value / bootstrap writes
//   warp  8     MMA issuer: tcgen05.mma M=128 N=256 K=16 in a fixed global
//               order, fp32 accumulators in TMEM (actor cols 0-255, critic 256-511)
//   warps 9+    producers (kProducers) of the weight ring
// Per net and step: 18 chunks = W1 [256x16] | W2 8 x [256x32] | W3 8 x [256x32] | W4 [16x256].
#include <cuda_bf16.h>

#include "pm_env.cuh"
#include "prb_internal.h"
#include "rng.cuh"
#include "rollout_pm_tc.h"
#include "tc.cuh"
#include "tmap.h"

namespace prb {
namespace {

constexpr int kM = 128;      // envs per tile == MMA M == TMEM lanes
constexpr int kHid = 256;    // hidden width
constexpr int kX = 16;       // obs tile width (6 used)
constexpr int kKC = kPmChunkK;         // K per weight chunk of the hidden layers
constexpr int kCPL = kHid / kKC;        // chunks per hidden layer
constexpr int kSlot = kHid * kKC * 2;   // bytes per chunk / ring slot ([256 N][kKC K] bf16)
constexpr int kStages = kKC == 16 ? 10 : 5;  // ring slots shared by both nets (smem: kStages x kSlot)
constexpr int kChunks = 2 + 2 * kCPL;   // chunks per net per step: W1 | W2 | W3 | W4
constexpr uint32_t kNetPack = kChunks * kSlot;
// W1 [256][16] and W4 [16][256] are 8 KB; the hidden-layer chunks are kSlot
__host__ __device__ constexpr uint32_t chunk_bytes(int c) { return (c == 0 || c == kChunks - 1) ? 8192u : (uint32_t)kSlot; }
__device__ __forceinline__ int op_nchunks(int layer) { return (layer == 1 || layer == 2) ? kCPL : 1; }
__device__ __forceinline__ int op_chunk(int layer, int q) {
  return layer == 0 ? 0 : (layer == 3 ? kChunks - 1 : 1 + kCPL * (layer - 1) + q);
}
constexpr int kProducers = 3;  // producer warps: one warp keeps ~one bulk copy in flight
constexpr int kThreads = 32 * (9 + kProducers);
// op k of a step: (net, layer) in issue order, see the kernel
__device__ constexpr int kOpNet[8] = {0, 1, 1, 0, 1, 0, 1, 0};
__device__ constexpr int kOpLayer[8] = {0, 3, 0, 1, 1, 2, 2, 3};
constexpr uint32_t kTmemCols = 512;
constexpr float kLogTwoPiF = 1.8378770664093454836f;
static_assert(2 * kNetPack == kPmPackBytes, "pack size");

// bf16 pack of the flat fp32 params in consumption order (B[n][k] = W[k][n]).
// Per net, 34 chunks of 8 KB: W1 [256][16], W2/W3 as 16 K-steps [256][16], W4 [16][256].
__global__ void pm_pack_kernel(const float* __restrict__ P, PmPackOffsets o, uint8_t* __restrict__ pack) {
  constexpr int kPerNet = 4096 + 2 * 65536 + 4096;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * kPerNet) return;
  const int net = i / kPerNet, j = i % kPerNet;
  const int* w = net ? o.c_w : o.a_w;
  uint8_t* base = pack + (size_t)net * kNetPack;
  float v;
  uint32_t off;
  if (j < 4096) {  // W1 [S x 256]
    const int n = j / kX, k = j % kX;
    v = (k < o.S) ? P[w[0] + k * kHid + n] : 0.f;
    off = tc::kmajor_offset(n, k, kX);
  } else if (j < 4096 + 2 * 65536) {  // W2 / W3 [256 x 256]
    const int jj = j - 4096, L = jj / 65536, r = jj % 65536, n = r / kHid, k = r % kHid;
    v = P[w[1 + L] + k * kHid + n];
    off = (uint32_t)(1 + kCPL * L + k / kKC) * kSlot + tc::kmajor_offset(n, k % kKC, kKC);
  } else {  // W4 [256 x out] -> [16][256]
    const int jj = j - 4096 - 2 * 65536, n = jj / kHid, k = jj % kHid;
    const int out = net ? 1 : o.A;
    v = (n < out) ? P[w[3] + k * out + n] : 0.f;
    off = (uint32_t)(kChunks - 1) * kSlot + tc::kmajor_offset(n, k, kHid);
  }
  *reinterpret_cast<__nv_bfloat16*>(base + off) = __float2bfloat16_rn(v);
}

// kPair: one CTA pair (cluster of 2 SMs) per 256 envs with cta_group::2 MMAs (M = 256).  Each
// CTA keeps its own 128 rows of A (obs / hidden tiles) and streams HALF of every weight chunk
// (the B columns n in [128·rank, 128·rank + 128), a contiguous half of the chunk's K-major
// image): the per-SM weight bytes halve while the per-SM MMA work is unchanged, which is what
// bounded the single-CTA kernel (profiles/mb/mb_l2smem.cu).  The leader (rank 0) issues every
// MMA; commits are multicast to both CTAs' barriers; the peer's epilogue groups arrive on the
// leader's barriers through DSMEM, and both CTAs' halves of a weight chunk are loaded by
// .cta_group::2 tensor-map TMA that completes on the leader's `full` barrier.
template <bool kPair>
struct PmCfg {
  static constexpr int kSlotB = kPair ? kSlot / 2 : kSlot;       // bytes per ring slot
  static constexpr int kStagesT = kPair ? 2 * kStages : kStages;  // same ring bytes
  static constexpr int kRows = kPair ? 2 * kM : kM;               // envs per (pair-)tile
  static constexpr uint32_t kArr = kPair ? 8 : 4;                 // epilogue-warp arrivals per signal
  // half-size copies complete no faster than whole ones (~350 clk each, one in flight per warp),
  // so a pair CTA keeps twice as many in flight
  static constexpr int kProd = kPair ? 2 * kProducers : kProducers;
  static constexpr int kThr = 32 * (9 + kProd);
};

template <bool kPair>
struct PmSmem {
  alignas(1024) uint8_t ring[PmCfg<kPair>::kStagesT][PmCfg<kPair>::kSlotB];  // weight ring (global op order)
  alignas(1024) uint8_t h[2][kM * kHid * 2];      // bf16 A operands [128][256]: actor, critic
  alignas(1024) uint8_t x[kM * kX * 2];           // bf16 obs tile [128][16]
  float bias[2][3][kHid];                         // hidden-layer biases [net][layer]
  float b4a[2], b4c, sig[2], isig[2], lpc;
  uint64_t full[PmCfg<kPair>::kStagesT], empty[PmCfg<kPair>::kStagesT];
  uint64_t dfull[2];  // MMA -> group: layer result in TMEM
  uint64_t ready[2];  // group -> MMA: operand written / accumulator free (epilogue-warp arrivals)
  uint64_t xready;    // actor group -> MMA: obs tile written
  uint64_t xfree;     // critic MMA -> actor group: the critic's L1 has consumed the obs tile
  uint64_t aepi1;     // actor group -> critic MMA: actor layer-1 epilogue done (phase offset)
  uint32_t tmem;
};

// clock64 event trace of CTA 0 (debug; a.trace == nullptr in production)
struct Tracer {
  unsigned long long* p = nullptr;
  int n = 0;
  __device__ __forceinline__ void mark() {
    if (p && n < kPmTraceLen) p[n++] = clock64();
  }
};

// one arrive per warp on the MMA issuer's barrier (the leader's, through DSMEM, in the peer)
template <bool kPair>
__device__ __forceinline__ void arrive_mma(uint64_t* bar, uint32_t rank) {
  if (kPair && rank != 0)
    tc::mbar_arrive_cluster(tc::mapa_shared(bar, 0));
  else
    tc::mbar_arrive(bar);
}

template <bool kPair>
__device__ __forceinline__ void group_signal(uint64_t* bar, uint32_t rank) {
  tc::fence_proxy_async();  // this thread's operand stores -> async proxy
  tc::fence_before_sync();  // this thread's TMEM loads are complete
  __syncwarp();
  if ((threadIdx.x & 31) == 0) arrive_mma<kPair>(bar, rank);
}

template <bool kPair>
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t ph) {
  if (kPair)
    tc::mbar_wait_cluster(bar, ph);
  else
    tc::mbar_wait(bar, ph);
}

template <bool kPair>
__device__ __forceinline__ void group_wait(uint64_t* bar, uint32_t& ph) {
  bar_wait<kPair>(bar, ph);
  ph ^= 1;
  tc::fence_after_sync();
}

// this thread's row of a 256-column accumulator -> tanh(. + b) -> bf16 operand row
__device__ __forceinline__ void epi_hidden(uint32_t trow, const float* bias, uint8_t* hb, int row) {
#pragma unroll 1
  for (int c = 0; c < kHid; c += 32) {
    uint32_t v[32];
    tc::tmem_ld32(trow + c, v);
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float z0 = __uint_as_float(v[2 * i]), z1 = __uint_as_float(v[2 * i + 1]);
      tc::add2(z0, z1, bias[c + 2 * i], bias[c + 2 * i + 1]);
      pk[i] = tc::pack_bf16(tc::tanh_fast(z0), tc::tanh_fast(z1));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<uint4*>(hb + tc::arow_offset(row, c + 8 * q)) =
          make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
}

template <bool kPair>
__global__ void __launch_bounds__(PmCfg<kPair>::kThr, 1) pm_rollout_tc_kernel(const __grid_constant__ PmTcArgs a) {
  using Cfg = PmCfg<kPair>;
  constexpr int kSlotB = Cfg::kSlotB, kStagesT = Cfg::kStagesT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  PmSmem<kPair>& s = *reinterpret_cast<PmSmem<kPair>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = kPair ? tc::cluster_ctarank() : 0u;
  const int unit = kPair ? (int)blockIdx.x / 2 : (int)blockIdx.x;     // pair (or CTA) index
  const int nunits = kPair ? (int)gridDim.x / 2 : (int)gridDim.x;
  const int ntiles = (a.N + Cfg::kRows - 1) / Cfg::kRows;
  const float* P = a.params;

  for (int i = tid; i < 2 * 3 * kHid; i += Cfg::kThr) {
    const int net = i / (3 * kHid), L = (i / kHid) % 3, n = i % kHid;
    const int w = net ? a.o.c_w[L] : a.o.a_w[L];
    const int in = (L == 0) ? a.o.S : kHid;
    s.bias[net][L][n] = P[w + in * kHid + n];
  }
  if (tid < 2) {
    s.b4a[tid] = P[a.o.a_w[3] + kHid * 2 + tid];
    const float l = P[a.o.log_std + tid];
    s.sig[tid] = expf(l);
    s.isig[tid] = expf(-l);
  }
  if (tid == 0) {
    s.b4c = P[a.o.c_w[3] + kHid];
    s.lpc = -kLogTwoPiF - P[a.o.log_std] - P[a.o.log_std + 1];
    for (int i = 0; i < kStagesT; ++i) {
      tc::mbar_init(&s.full[i], 1);
      tc::mbar_init(&s.empty[i], 1);
    }
    for (int n = 0; n < 2; ++n) {
      tc::mbar_init(&s.dfull[n], 1);
      tc::mbar_init(&s.ready[n], Cfg::kArr);
    }
    tc::mbar_init(&s.xready, Cfg::kArr);
    tc::mbar_init(&s.xfree, 1);
    tc::mbar_init(&s.aepi1, Cfg::kArr);
  }
  if (warp == 8) {
    if (kPair)
      tc::tmem_alloc_pair(&s.tmem, kTmemCols);
    else
      tc::tmem_alloc(&s.tmem, kTmemCols);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (kPair) tc::cluster_sync();  // both CTAs' barriers initialised before any DSMEM arrive
  tc::fence_after_sync();
  const uint32_t tbase = s.tmem;

  // Global MMA order, identical for the producers and the issuer.  Per step g:
  //   A1(g), C4(g-1), C1(g), A2(g), C2(g), A3(g), C3(g), A4(g)      and a final C4.
  // The critic runs about one epilogue behind the actor (C1 waits for the actor's
  // layer-1 epilogue), so this order is also the order in which the operands
  // become ready: one ring serves both nets without head-of-line blocking.
  const int my_tiles = (ntiles - unit + nunits - 1) / nunits;
  const int G = my_tiles * (a.H + 1);  // steps this CTA (pair) runs
  // every chunk of the global order, in order: f(it, net, chunk)
  auto for_each_chunk = [&](auto&& f) {
    uint32_t it = 0;
    for (int g = 0; g <= G; ++g)
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        if ((g == G && k != 1) || (g == 0 && k == 1)) continue;
        const int net = kOpNet[k], layer = kOpLayer[k], nq = op_nchunks(layer);
#pragma unroll 1
        for (int q = 0; q < nq; ++q, ++it) f(it, net, op_chunk(layer, q));
      }
  };
  if (warp >= 9) {  // ---------------- producers ----------------
    // Bulk copies issued by one warp complete roughly one at a time
    // (profiles/mb/mb_l2smem.cu); chunk `it` goes to producer it % kProd.
    const int pr = warp - 9;
    if (lane == 0) {
      for_each_chunk([&](uint32_t it, int net, int c) {
        if ((int)(it % Cfg::kProd) != pr) return;
        const uint32_t slot = it % kStagesT, use = it / kStagesT;
        if (use) bar_wait<kPair>(&s.empty[slot], (use - 1) & 1);
        if constexpr (kPair) {
          // this CTA's half of chunk c: rows [off/256, +half/256) of the [.][128] bf16 view, 16-row boxes;
          // both halves complete on the leader's full[slot], which expects the whole chunk
          const uint32_t half = chunk_bytes(c) / 2;
          const uint32_t off = (uint32_t)net * kNetPack + (uint32_t)c * kSlot + rank * half;
          const uint32_t bar = tc::mapa_shared(&s.full[slot], 0);
          if (rank == 0) tc::mbar_arrive_expect_tx(&s.full[slot], 2 * half);
          for (uint32_t b = 0; b < half; b += 4096)
            tc::tma_load_2d_pair(s.ring[slot] + b, &a.pack_map, 0, (int)((off + b) >> 8), bar);
        } else {
          tc::mbar_arrive_expect_tx(&s.full[slot], chunk_bytes(c));
          tc::bulk_g2s(s.ring[slot], a.pack + (size_t)net * kNetPack + (size_t)c * kSlot, chunk_bytes(c),
                       &s.full[slot]);
        }
      });
    }
  } else if (warp == 8) {  // ---------------- MMA issuer (leader) / relay (peer) ----------------
    if (lane == 0 && rank == 0) {
      constexpr uint32_t ID_256 = tc::idesc_bf16(Cfg::kRows, kHid), ID_16 = tc::idesc_bf16(Cfg::kRows, 16);
      const uint32_t x_addr = tc::smem_u32(s.x), ring0 = tc::smem_u32(s.ring[0]);
      uint32_t it = 0, rph[2] = {0, 0}, xph = 0, eph = 0;
      Tracer tr;
      if (a.trace && blockIdx.x == 0) tr.p = a.trace + 2 * kPmTraceLen;
      unsigned long long waited = 0;  // trace: clocks spent waiting for weight chunks
      auto take = [&]() -> uint32_t {  // next weight chunk: wait until it (both halves) has landed
        const uint32_t slot = it % kStagesT, ph = (it / kStagesT) & 1;
        const unsigned long long t0 = tr.p ? clock64() : 0ull;
        bar_wait<kPair>(&s.full[slot], ph);  // both halves (pair: the peer's TMA completes here too)
        if (tr.p) waited += clock64() - t0;
        return ring0 + slot * kSlotB;
      };
      auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
        if (kPair)
          tc::mma_bf16_pair(d, ad, bd, id, acc);
        else
          tc::mma_bf16(d, ad, bd, id, acc);
      };
      auto commit = [&](uint64_t* bar) {
        if (kPair)
          tc::mma_commit_pair(bar);
        else
          tc::mma_commit(bar);
      };
      auto release = [&]() {  // the chunk's MMAs done -> slot reusable (in both CTAs)
        commit(&s.empty[it % kStagesT]);
        ++it;
      };
      for (int g = 0; g <= G; ++g)
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
          if ((g == G && k != 1) || (g == 0 && k == 1)) continue;
          const int net = kOpNet[k], layer = kOpLayer[k];
          if (net == 0 && layer == 0) {
            bar_wait<kPair>(&s.xready, xph);  // obs tile written
            xph ^= 1;
          } else {
            bar_wait<kPair>(&s.ready[net], rph[net]);  // operand written / accumulator read
            rph[net] ^= 1;
            if (net == 1 && layer == 0) {  // the actor's layer-1 epilogue is done (phase offset)
              bar_wait<kPair>(&s.aepi1, eph);
              eph ^= 1;
            }
          }
          tc::fence_after_sync();
          tr.mark();
          const uint32_t d = tbase + (uint32_t)net * kHid;
          const uint32_t h_addr = tc::smem_u32(s.h[net]);
          // B operands: [n][k] K-major; in pair mode each CTA's slot holds its n-half, same strides
          if (layer == 0) {  // [128 x 16] obs . [16 x 256]
            const uint32_t b = take();
            mma(d, tc::smem_desc(x_addr, 2048, 128), tc::smem_desc(b, 128, kX * 16), ID_256, 0);
            release();
            if (net == 1) commit(&s.xfree);
          } else if (layer < 3) {  // [128 x 256] h . [256 x 256], kCPL chunks of kKC/16 K-steps
#pragma unroll 1
            for (int q = 0; q < kCPL; ++q) {
              const uint32_t b = take();
#pragma unroll
              for (int j = 0; j < kKC / 16; ++j)
                mma(d, tc::smem_desc(h_addr + (q * (kKC / 16) + j) * 4096, 2048, 128),
                    tc::smem_desc(b + j * 256, 128, kKC * 16), ID_256, (q | j) != 0);
              release();
            }
          } else {  // head: [128 x 256] h . [256 x 16]
            const uint32_t b = take();
#pragma unroll
            for (int j = 0; j < 16; ++j)
              mma(d, tc::smem_desc(h_addr + j * 4096, 2048, 128), tc::smem_desc(b + j * 256, 128, kHid * 16),
                  ID_16, j != 0);
            release();
          }
          commit(&s.dfull[net]);
          tr.mark();
          if (tr.p && g < 8 && k == 7) a.trace[3 * kPmTraceLen + g] = waited;
        }
    }
  } else if (warp < 4) {  // ---------------- actor group ----------------
    const int row = tid;
    const uint32_t trow = tbase + ((uint32_t)(warp * 32) << 16);
    uint32_t dph = 0, fph = 0;
    bool first = true;
    Tracer tr;
    if (a.trace && blockIdx.x == 0 && tid == 0) tr.p = a.trace;
    const size_t N = a.N;
    for (int tile = unit; tile < ntiles; tile += nunits) {
      const size_t e = (size_t)tile * Cfg::kRows + rank * kM + row;
      const bool live = e < N;
      double st[6];
      int32_t steps = 0, idx = 0;
      double ret = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) st[j] = live ? a.st[j * N + e] : 0.0;
      if (live) {
        steps = a.steps[e];
        ret = a.ep_return[e];
        idx = a.mt_idx[e];
      }
      for (int h = 0; h <= a.H; ++h) {
        float o[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) o[j] = (float)st[j];
        if (!first) {  // the critic's L1 of the previous step has consumed X
          bar_wait<kPair>(&s.xfree, fph);
          fph ^= 1;
        }
        first = false;
        {  // obs row -> X (bf16, cols 6..15 zero)
          *reinterpret_cast<uint4*>(s.x + tc::arow_offset(row, 0)) =
              make_uint4(tc::pack_bf16(o[0], o[1]), tc::pack_bf16(o[2], o[3]), tc::pack_bf16(o[4], o[5]), 0u);
          *reinterpret_cast<uint4*>(s.x + tc::arow_offset(row, 8)) = make_uint4(0u, 0u, 0u, 0u);
        }
        group_signal<kPair>(&s.xready, rank);
        tr.mark();
#pragma unroll 1
        for (int L = 0; L < 3; ++L) {
          group_wait<kPair>(&s.dfull[0], dph);
          tr.mark();
          epi_hidden(trow, s.bias[0][L], s.h[0], row);
          group_signal<kPair>(&s.ready[0], rank);
          if (L == 0 && (threadIdx.x & 31) == 0) arrive_mma<kPair>(&s.aepi1, rank);
          tr.mark();
        }
        group_wait<kPair>(&s.dfull[0], dph);
        tr.mark();
        float mv[16];
        tc::tmem_ld16(trow, mv);
        if (h == a.H) {  // the VecEnv's states after the rollout
          if (live)
#pragma unroll
            for (int j = 0; j < 6; ++j) a.obs_out[e * 6 + j] = o[j];
          break;
        }
        // a = mu + sigma * eps (Philox stream of policy_kernel), log-prob (nn.hpp:215-224,250-265)
        const Philox4 rr = philox4x32_10((uint32_t)a.seed, (uint32_t)(a.seed >> 32), 0u, (uint32_t)e, (uint32_t)h, 0u);
        const float2 z = box_muller(rr.x, rr.y);
        const float m0 = mv[0] + s.b4a[0], m1 = mv[1] + s.b4a[1];
        const float act0 = m0 + s.sig[0] * z.x, act1 = m1 + s.sig[1] * z.y;
        const float z0 = (act0 - m0) * s.isig[0], z1 = (act1 - m1) * s.isig[1];
        const float lp = s.lpc - 0.5f * (z0 * z0 + z1 * z1);
        // VecEnv step: clamp to the spec bounds (env.hpp:213-215), pointmass_step, auto-reset
        double n[6], r;
        bool done;
        pm::step(st, pm::clamp_ref((double)act0, -1.0, 1.0), pm::clamp_ref((double)act1, -1.0, 1.0), steps, n, r,
                 done);
        ret = __dadd_rn(ret, r);
        if (done) {
          if (live) pm::reset_draws(a.mt + e, N, idx, n);
          steps = 0;
          ret = 0.0;
        } else {
          ++steps;
        }
        if (live) {
          const size_t slab = (size_t)h * N + e;
          float2* ob = reinterpret_cast<float2*>(a.b_obs + slab * 6);
          ob[0] = make_float2(o[0], o[1]);
          ob[1] = make_float2(o[2], o[3]);
          ob[2] = make_float2(o[4], o[5]);
          reinterpret_cast<float2*>(a.b_act)[slab] = make_float2(act0, act1);
          a.b_logp[slab] = lp;
          a.b_rew[slab] = (float)r;
          a.b_done[slab] = done ? 1 : 0;
        }
#pragma unroll
        for (int j = 0; j < 6; ++j) st[j] = n[j];
        tr.mark();
      }
      if (live) {
#pragma unroll
        for (int j = 0; j < 6; ++j) a.st[j * N + e] = st[j];
        a.steps[e] = steps;
        a.ep_return[e] = ret;
        a.mt_idx[e] = idx;
      }
    }
  } else {  // ---------------- critic group (warps 4-7) ----------------
    const int row = tid - kM;
    const uint32_t trow = tbase + ((uint32_t)((warp - 4) * 32) << 16) + kHid;
    uint32_t dph = 0;
    Tracer tr;
    if (a.trace && blockIdx.x == 0 && tid == kM) tr.p = a.trace + kPmTraceLen;
    const size_t N = a.N;
    group_signal<kPair>(&s.ready[1], rank);  // critic accumulator free
    for (int tile = unit; tile < ntiles; tile += nunits) {
      const size_t e = (size_t)tile * Cfg::kRows + rank * kM + row;
      const bool live = e < N;
      for (int h = 0; h <= a.H; ++h) {
#pragma unroll 1
        for (int L = 0; L < 3; ++L) {
          group_wait<kPair>(&s.dfull[1], dph);
          tr.mark();
          epi_hidden(trow, s.bias[1][L], s.h[1], row);
          group_signal<kPair>(&s.ready[1], rank);
          tr.mark();
        }
        group_wait<kPair>(&s.dfull[1], dph);
        tr.mark();
        float vv[16];
        tc::tmem_ld16(trow, vv);
        group_signal<kPair>(&s.ready[1], rank);  // accumulator read: the next step's L1 may overwrite it
        const float value = vv[0] + s.b4c;
        tr.mark();
        if (live) {
          if (h == a.H)
            a.b_boot[e] = value;  // bootstrap V(s_H) (pod.hpp:127-131)
          else
            a.b_val[(size_t)h * N + e] = value;
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (kPair) tc::cluster_sync();  // the peer is done with TMEM and DSMEM before the pair deallocates
  if (warp == 8) {
    if (kPair)
      tc::tmem_dealloc_pair(tbase, kTmemCols);
    else
      tc::tmem_dealloc(tbase, kTmemCols);
  }
}

}  // namespace

size_t pm_rollout_tc_smem() { return sizeof(PmSmem<true>) > sizeof(PmSmem<false>) ? sizeof(PmSmem<true>) : sizeof(PmSmem<false>); }

void launch_pm_pack(const float* params, const PmPackOffsets& o, uint8_t* pack, cudaStream_t s) {
  const int total = 2 * (4096 + 2 * 65536 + 4096);
  pm_pack_kernel<<<(total + 255) / 256, 256, 0, s>>>(params, o, pack);
  PRB_CHECK_LAUNCH();
}

// The pack as a 2-D bf16 tensor [kPmPackBytes / 256 rows][128], boxes of [16 rows][128] = 4 KB
// (every half chunk is a whole number of boxes).
void encode_pm_pack_map(CUtensorMap* map, const uint8_t* pack) {
  encode_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, pack, 128, kPmPackBytes / 256, 256, 128, 16);
}

// PRB_PM_PAIR=1 selects the CTA-pair kernel; the single-CTA kernel is the default because it is
// faster: 1.37e9 vs 1.13e9 transitions/s at configs[2].  The pair halves the
// per-SM weight bytes, but the layer time was not bound by them: each M=256 pair MMA takes as
// long as an M=128 single one (same per-SM tensor throughput), the epilogues are bound by the
// 16/clk/SM MUFU tanh rate, and every epilogue -> MMA hand-off now crosses SMs.
void launch_pm_rollout_tc(const PmTcArgs& a, int num_sms, cudaStream_t s) {
  const bool pair = debug_option(PRB_OPT_PM_CTA_PAIR) != 0;  // tests: the opt-in CTA-pair kernel
  ensure_smem(pm_rollout_tc_kernel<false>, sizeof(PmSmem<false>));
  ensure_smem(pm_rollout_tc_kernel<true>, sizeof(PmSmem<true>));
  if (pair) {
    PmTcArgs ap = a;
    encode_pm_pack_map(&ap.pack_map, a.pack);
    const int ntiles = (a.N + 2 * kM - 1) / (2 * kM);
    const int npairs = ntiles < num_sms / 2 ? ntiles : num_sms / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * npairs);
    cfg.blockDim = dim3(PmCfg<true>::kThr);
    cfg.dynamicSmemBytes = sizeof(PmSmem<true>);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PRB_CUDA(cudaLaunchKernelEx(&cfg, pm_rollout_tc_kernel<true>, ap));
  } else {
    const int ntiles = (a.N + kM - 1) / kM;
    const int grid = ntiles < num_sms ? ntiles : num_sms;
    pm_rollout_tc_kernel<false><<<grid, PmCfg<false>::kThr, sizeof(PmSmem<false>), s>>>(a);
  }
  PRB_CHECK_LAUNCH();
}

}  // namespace prb
