// zo2_common.cuh -- shared definitions for the sm_100a ZO2 step library.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include "../../include/zo2b200.h"

#define ZO2_CHECK_LAUNCH()                                   \
  do {                                                       \
    cudaError_t e__ = cudaGetLastError();                    \
    if (e__ != cudaSuccess) return zo2_set_cuda_error(e__);  \
  } while (0)

#define ZO2_CUDA_TRY(x)                                      \
  do {                                                       \
    cudaError_t e__ = (x);                                   \
    if (e__ != cudaSuccess) return zo2_set_cuda_error(e__);  \
  } while (0)

int zo2_set_cuda_error(cudaError_t e);
int zo2_set_error(int code, const char *msg);

static inline unsigned zo2_grid_for(uint64_t work, unsigned per_block,
                                    unsigned cap = 148u * 32u) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}
