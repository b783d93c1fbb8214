// Small layout / reduction helpers used around the router GEMMs.
//   * router weight staging: W_r [h, E] -> W_r^T padded [Epad, h] (logits GEMM B operand,
//     K-major) and W_r padded [h, Epad] (router dX GEMM B operand).
//   * deterministic fixed-order reduction of split-K fp32 partials (router dW_r).
#include "common.cuh"

namespace moe {
namespace util {

__global__ void stage_router_weight_kernel(const __nv_bfloat16* __restrict__ w, int h, int E,
                                           int Epad, __nv_bfloat16* __restrict__ wt_pad,
                                           __nv_bfloat16* __restrict__ w_pad) {
  const long long n = (long long)h * Epad;
  const __nv_bfloat16 zero = __float2bfloat16_rn(0.f);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / Epad);  // h index
    const int c = (int)(i % Epad);  // expert index
    const __nv_bfloat16 v = c < E ? w[(long long)r * E + c] : zero;
    if (w_pad) w_pad[i] = v;
    if (wt_pad) wt_pad[(long long)c * h + r] = v;
  }
}

// out[r, c] = sum_g in[g, r, c] for c < cols_out (in row stride cols_in); g ascending.
__global__ void reduce_groups_kernel(const float* __restrict__ in, int G, int rows, int cols_in,
                                     int cols_out, float* __restrict__ out) {
  const long long n = (long long)rows * cols_out;
  const long long gs = (long long)rows * cols_in;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols_out), c = (int)(i % cols_out);
    float s = 0.f;
    for (int g = 0; g < G; ++g) s += in[g * gs + (long long)r * cols_in + c];
    out[i] = s;
  }
}

}  // namespace util
}  // namespace moe

using namespace moe;

extern "C" {

int moe_stage_router_weight(const void* w, int h, int E, int Epad, void* wt_pad, void* w_pad,
                            void* stream) {
  if (E > Epad) return kErrInvalidArg;
  util::stage_router_weight_kernel<<<1024, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(w), h, E, Epad, static_cast<__nv_bfloat16*>(wt_pad),
      static_cast<__nv_bfloat16*>(w_pad));
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_reduce_groups_f32(const float* in, int G, int rows, int cols_in, int cols_out, float* out,
                          void* stream) {
  util::reduce_groups_kernel<<<1024, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      in, G, rows, cols_in, cols_out, out);
  MOE_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"
