// mlp_simt.cuh -- fp32 SIMT building blocks for the MLP forward/backward of
// the actor and critic (nn.hpp:63-132) on a tile of rows resident in shared
// memory.  Weights are in the reference layout W[in][out] row-major with a
// row stride `ldw` (== out in HBM; out+1 when staged into shared memory so
// both row- and column-wise walks are bank-conflict free).
#pragma once
#include <cstdint>

namespace prb {

constexpr int kMaxLayers = 8;

struct MlpDesc {
  int nl;                    // number of linear layers
  int dims[kMaxLayers + 1];  // dims[0] = input, dims[nl] = output
  int off[kMaxLayers];       // flat offset of W_i (b_i follows at off + in*out)
};

// Where each layer's weights / biases live for one kernel (HBM or staged smem).
struct LayerPtrs {
  const float* W[kMaxLayers];
  const float* B[kMaxLayers];
  int ldw[kMaxLayers];
};

__device__ __forceinline__ int round4(int x) { return (x + 3) & ~3; }

// s_out[r][j] = act(sum_k s_in[r][k] W[k][j] + b[j]) for r < nrows.
// Thread mapping: column j = tid % TJ (TJ = pow2 >= min(out, blockDim)), row
// group g = tid / TJ owning RB consecutive rows per pass.  ldi is a multiple
// of 4; smem tiles have at least round8(nrows) rows.
template <bool TANH, int RB>
__device__ __forceinline__ void linear_tile_rb(const float* __restrict__ W, int ldw, const float* __restrict__ b,
                                               int in, int out, const float* s_in, int ldi, float* s_out, int ldo,
                                               int nrows, int TJ) {
  const int G = blockDim.x / TJ;
  const int tj = threadIdx.x % TJ, g = threadIdx.x / TJ;
  const int in4 = in & ~3;
  for (int j0 = 0; j0 < out; j0 += TJ) {
    const int j = j0 + tj;
    if (j >= out) continue;
    const float bj = b[j];
    for (int rb = g * RB; rb < nrows; rb += G * RB) {
      float acc[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) acc[i] = 0.0f;
      int k = 0;
      for (; k < in4; k += 4) {
        const float w0 = W[(size_t)(k + 0) * ldw + j];
        const float w1 = W[(size_t)(k + 1) * ldw + j];
        const float w2 = W[(size_t)(k + 2) * ldw + j];
        const float w3 = W[(size_t)(k + 3) * ldw + j];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          const float4 x = *reinterpret_cast<const float4*>(s_in + (rb + i) * ldi + k);
          acc[i] = fmaf(x.x, w0, acc[i]);
          acc[i] = fmaf(x.y, w1, acc[i]);
          acc[i] = fmaf(x.z, w2, acc[i]);
          acc[i] = fmaf(x.w, w3, acc[i]);
        }
      }
      for (; k < in; ++k) {
        const float w = W[(size_t)k * ldw + j];
#pragma unroll
        for (int i = 0; i < RB; ++i) acc[i] = fmaf(s_in[(rb + i) * ldi + k], w, acc[i]);
      }
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        if (rb + i < nrows) {
          const float z = acc[i] + bj;
          s_out[(rb + i) * ldo + j] = TANH ? tanhf(z) : z;
        }
      }
    }
  }
}

template <bool TANH>
__device__ __forceinline__ void linear_tile(const float* __restrict__ W, int ldw, const float* __restrict__ b, int in,
                                            int out, const float* s_in, int ldi, float* s_out, int ldo, int nrows) {
  int TJ = 32;
  while (TJ < out && TJ < (int)blockDim.x) TJ <<= 1;
  const int G = blockDim.x / TJ;
  // rows per thread per pass: the smallest RB whose G x RB rows cover the tile in ONE pass (each
  // pass re-walks the weights: for a few rows the walk's load latency is the whole cost), else 8.
  // A row's sum is the same fmaf chain over k whatever RB is.
  if (nrows > 4 * G)
    linear_tile_rb<TANH, 8>(W, ldw, b, in, out, s_in, ldi, s_out, ldo, nrows, TJ);
  else if (nrows > 2 * G)
    linear_tile_rb<TANH, 4>(W, ldw, b, in, out, s_in, ldi, s_out, ldo, nrows, TJ);
  else if (nrows > G)
    linear_tile_rb<TANH, 2>(W, ldw, b, in, out, s_in, ldi, s_out, ldo, nrows, TJ);
  else
    linear_tile_rb<TANH, 1>(W, ldw, b, in, out, s_in, ldi, s_out, ldo, nrows, TJ);
}

// Forward through all layers with explicit weight locations.  acts[l] (ld
// lds[l]) receives layer l's post-activation output; s_x is the input.
__device__ __forceinline__ void mlp_forward_tile_p(const MlpDesc& d, const LayerPtrs& lp, const float* s_x, int ldx,
                                                   float* const* acts, const int* lds, int nrows) {
  const float* in = s_x;
  int ldi = ldx;
  for (int l = 0; l < d.nl; ++l) {
    if (l + 1 < d.nl)
      linear_tile<true>(lp.W[l], lp.ldw[l], lp.B[l], d.dims[l], d.dims[l + 1], in, ldi, acts[l], lds[l], nrows);
    else
      linear_tile<false>(lp.W[l], lp.ldw[l], lp.B[l], d.dims[l], d.dims[l + 1], in, ldi, acts[l], lds[l], nrows);
    __syncthreads();
    in = acts[l];
    ldi = lds[l];
  }
}

// Forward with the weights read straight from the flat blob in HBM/L2.
__device__ __forceinline__ void mlp_forward_tile(const float* __restrict__ params, const MlpDesc& d, const float* s_x,
                                                 int ldx, float* const* acts, const int* lds, int nrows) {
  LayerPtrs lp;
  for (int l = 0; l < d.nl; ++l) {
    lp.W[l] = params + d.off[l];
    lp.B[l] = lp.W[l] + (size_t)d.dims[l] * d.dims[l + 1];
    lp.ldw[l] = d.dims[l + 1];
  }
  mlp_forward_tile_p(d, lp, s_x, ldx, acts, lds, nrows);
}

}  // namespace prb
