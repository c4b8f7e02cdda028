// ph_kernels.h — internal launcher interface between the C ABI (ph_abi.cu)
// and the kernels (ph_query.cu, ph_query_bytes.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ph_device.cuh"

namespace phg {

cudaError_t launch_query_u64(const DevIndex& ix, int gamma_kind, bool pow2, const uint64_t* keys,
                             void* out, int out_width, uint64_t n, int minimal, cudaStream_t s,
                             int sms);

cudaError_t launch_query_bytes(const DevIndex& ix, int gamma_kind, bool pow2,
                               const uint8_t* bytes, const uint64_t* offsets, uint64_t base_off,
                               void* out, int out_width, uint64_t n, int minimal, cudaStream_t s,
                               int sms);

uint64_t launch_count();
void note_launch();
void set_launch(int threads, int bps);

}  // namespace phg
