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

// HBM write-only probes (bench.py's write bound for write-dominated kernels). Zeros written
// over `bytes` (a multiple of 16). mode 0: 16-byte stores, 4 in flight per thread; mode 1:
// the same with .cs (streaming) stores; mode 2: TMA bulk stores of a zeroed 32 KB smem chunk
// (one issuing thread per CTA, up to 8 groups in flight).
constexpr int kProbeChunk = 32768;

template <bool CS>
__global__ void __launch_bounds__(512) write_probe_st_kernel(uint4* __restrict__ dst,
                                                             long long n16) {
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if constexpr (CS) __stcs(dst + i + u * stride, z);
      else dst[i + u * stride] = z;
    }
  }
  for (; i < n16; i += stride) dst[i] = z;
}

__global__ void __launch_bounds__(32) write_probe_bulk_kernel(char* __restrict__ dst,
                                                              long long bytes) {
  extern __shared__ __align__(128) uint4 zbuf[];
  for (int i = threadIdx.x; i < kProbeChunk / 16; i += blockDim.x)
    zbuf[i] = make_uint4(0u, 0u, 0u, 0u);
  fence_async_shared();
  __syncwarp();
  if (threadIdx.x != 0) return;
  const long long chunks = bytes / kProbeChunk;
  int inflight = 0;
  for (long long c = blockIdx.x; c < chunks; c += gridDim.x) {
    bulk_store_s2g(dst + c * kProbeChunk, zbuf, kProbeChunk);
    bulk_commit();
    if (++inflight >= 8) asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
  }
  const long long tail = bytes - chunks * kProbeChunk;  // multiple of 16
  if (blockIdx.x == 0 && tail > 0) {
    bulk_store_s2g(dst + chunks * kProbeChunk, zbuf, (uint32_t)tail);
    bulk_commit();
  }
  bulk_wait_all();
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

// bench.py's HBM write-only bandwidth probe: zeros `bytes` (multiple of 16) at dst.
int moe_hbm_write_probe(void* dst, long long bytes, int mode, void* stream) {
  if (!dst || bytes <= 0 || (bytes & 15) || ((uintptr_t)dst & 15) || mode < 0 || mode > 2)
    return kErrInvalidArg;
  auto st = static_cast<cudaStream_t>(stream);
  const int sms = device_sms();
  if (mode == 2) {
    util::write_probe_bulk_kernel<<<sms * 4, 32, util::kProbeChunk, st>>>(
        static_cast<char*>(dst), bytes);
  } else if (mode == 1) {
    util::write_probe_st_kernel<true><<<sms * 4, 512, 0, st>>>(static_cast<uint4*>(dst),
                                                                bytes / 16);
  } else {
    util::write_probe_st_kernel<false><<<sms * 4, 512, 0, st>>>(static_cast<uint4*>(dst),
                                                                 bytes / 16);
  }
  MOE_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"
