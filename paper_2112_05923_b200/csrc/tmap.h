// tmap.h -- host-side encoding of 2-D TMA tensor maps (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so libprb.so needs no -lcuda).
#pragma once

#include <cuda.h>

#include <cstdint>

namespace prb {

// A row-major [dim1][dim0] tensor of `dtype` at `base` (row pitch stride1_bytes, a multiple of
// 16), boxes of [box1][box0] elements, no swizzle, out-of-bounds elements zero-filled.
void encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, uint64_t dim0, uint64_t dim1,
                    uint64_t stride1_bytes, uint32_t box0, uint32_t box1,
                    CUtensorMapL2promotion l2 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B);

}  // namespace prb
