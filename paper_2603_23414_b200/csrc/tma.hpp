// tma.hpp — host-side TMA tensor-map encoding (driver entry point fetched at
// run time so the library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace srl {

// Returns 0 on success.  2-D bf16 (or fp32 when elem_bytes==4) row-major
// tensor [rows, cols] (cols contiguous), box [box_rows, box_cols], 128B swizzle
// when box_cols*elem_bytes == 128, otherwise no swizzle.
int tma_encode_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                  uint64_t row_stride_bytes, uint32_t box_rows, uint32_t box_cols, int elem_bytes,
                  bool swizzle128);

}  // namespace srl
