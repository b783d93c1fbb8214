// MXFP8 quantisation (1x32 blocks, E8M0 scales, E4M3 payload): the reference's MXFP8 recipe
// (pkg/src/moelab/quant.py:62-64, :166-201; formats.py:16-139) as one fused pass, producing
// both the payload codes and the scale factors in the tiled layout the block-scaled tcgen05
// GEMM stages through tcgen05.cp (csrc/grouped_gemm_mxfp8.cu).
//
// Bit-exact with the reference: scale = 2^ceil(log2(amax / 448)) from the exponent of amax
// (frexp, no log2 rounding), x * 2^-e is exact, and cvt.rn.satfinite.e4m3 is
// round-to-nearest-even on the E4M3 lattice (subnormals included) with saturation at 448.
#include <cuda_fp8.h>

#include "common.cuh"

namespace moe {
namespace mx {

// E8M0 exponent of a 1x32 block: smallest e with amax <= 448 * 2^e, clamped to [-127, 127].
__device__ __forceinline__ int e8m0_exp(float amax) {
  if (!(amax > 0.f)) return -127;
  int q;
  const float f = frexpf(amax, &q);  // amax = f * 2^q, f in [0.5, 1); 448 = 0.875 * 2^9
  int e = q - 9 + (f > 0.875f ? 1 : 0);
  return e < -127 ? -127 : (e > 127 ? 127 : e);
}

// Byte offset of (row, 32-block kb) in the tiled scale layout: per (128-row tile, 4-block
// K stage) a 512-byte chunk, byte i*16 + c*4 + j <- row tile*128 + c*32 + i, block stage*4+j.
__device__ __forceinline__ long long tiled_sf_offset(int row, int kb, int kblocks) {
  const int tile = row >> 7, rr = row & 127, c = rr >> 5, i = rr & 31;
  const int stage = kb >> 2, j = kb & 3;
  return ((long long)tile * (kblocks >> 2) + stage) * 512 + i * 16 + c * 4 + j;
}

// Input row of output row r when re-interleaving a stacked W1 [E, 2m, h] from the bf16
// engine's 128-row gate/up blocks to the MXFP8 engine's 64-row blocks (w1_m = m), else r.
__device__ __forceinline__ long long src_row(int r, int w1_m) {
  if (!w1_m) return r;
  const int two_m = 2 * w1_m;
  const int e = r / two_m, rr = r % two_m;
  const int j = rr >> 7, within = rr & 127;
  const int idx = 64 * j + (within & 63);  // gate / up index
  const int base = (idx >> 7) * 256 + (idx & 127);
  return (long long)e * two_m + base + (within >= 64 ? 128 : 0);
}

__global__ void quant_kernel(const __nv_bfloat16* __restrict__ x, long long ldx, int rows,
                             int K, uint8_t* __restrict__ codes, long long ldc,
                             uint8_t* __restrict__ sf_plain, uint8_t* __restrict__ sf_tiled,
                             int w1_m) {
  const int kblocks = K / 32;
  const long long n = (long long)rows * kblocks;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < n;
       id += (long long)gridDim.x * blockDim.x) {
    const int row = static_cast<int>(id / kblocks), kb = static_cast<int>(id % kblocks);
    const int4* src = reinterpret_cast<const int4*>(x + src_row(row, w1_m) * ldx + kb * 32);
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ld_nc_v4(src + u);
    float f[32];
    float amax = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[u]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 p = unpack_bf16x2(w[q]);
        f[u * 8 + 2 * q] = p.x;
        f[u * 8 + 2 * q + 1] = p.y;
        amax = fmaxf(amax, fmaxf(fabsf(p.x), fabsf(p.y)));
      }
    }
    const int e = e8m0_exp(amax);
    const float inv = __int_as_float((127 - e) << 23);  // 2^-e, e in [-127, 127] -> normal
    uint32_t out[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
          make_float2(f[4 * q] * inv, f[4 * q + 1] * inv), __NV_SATFINITE, __NV_E4M3);
      const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
          make_float2(f[4 * q + 2] * inv, f[4 * q + 3] * inv), __NV_SATFINITE, __NV_E4M3);
      out[q] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
    }
    int4* dst = reinterpret_cast<int4*>(codes + row * ldc + kb * 32);
    dst[0] = make_int4(out[0], out[1], out[2], out[3]);
    dst[1] = make_int4(out[4], out[5], out[6], out[7]);
    const uint8_t sc = static_cast<uint8_t>(e + 127);
    if (sf_plain) sf_plain[(long long)row * kblocks + kb] = sc;
    if (sf_tiled) sf_tiled[tiled_sf_offset(row, kb, kblocks)] = sc;
  }
}

// Transposing quantisation ("column twin", the reference's with_column_twin quant.py:195-200):
// x [B, R, C] bf16 -> codes [B, C, R] with 1x32 blocks along R, scales in the tiled layout
// of the [B*C, R] operand. A CTA handles 64 rows x 256 columns of one batch: the tile is
// staged in shared memory (8 x 16-byte loads in flight per thread), then thread c quantises
// column c's two 32-row blocks and writes them as one contiguous 64-byte run of the output
// row.
constexpr int QT_ROWS = 64;
__global__ void __launch_bounds__(256) quant_t_kernel(const __nv_bfloat16* __restrict__ x,
                                                      int B, int R, int C,
                                                      uint8_t* __restrict__ codes,
                                                      uint8_t* __restrict__ sf_tiled,
                                                      uint8_t* __restrict__ sf_plain) {
  __shared__ __nv_bfloat16 tile[QT_ROWS][256 + 8];
  const int cblocks = (C + 255) / 256, rblocks = R / QT_ROWS;
  const long long nt = (long long)B * rblocks * cblocks;
  for (long long id = blockIdx.x; id < nt; id += gridDim.x) {
    const int b = static_cast<int>(id / ((long long)rblocks * cblocks));
    const int rem = static_cast<int>(id % ((long long)rblocks * cblocks));
    const int rb = rem / cblocks, cb = rem % cblocks;
    const int r0 = rb * QT_ROWS, c0 = cb * 256;
    const __nv_bfloat16* src = x + ((long long)b * R + r0) * C + c0;
    int4 v[QT_ROWS * 32 / 256];
#pragma unroll
    for (int k = 0; k < QT_ROWS * 32 / 256; ++k) {
      const int i = threadIdx.x + k * 256;
      const int r = i / 32, q = i % 32;
      v[k] = c0 + q * 8 < C ? ld_nc_v4(src + (long long)r * C + q * 8) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < QT_ROWS * 32 / 256; ++k) {
      const int i = threadIdx.x + k * 256;
      *reinterpret_cast<int4*>(&tile[i / 32][(i % 32) * 8]) = v[k];
    }
    __syncthreads();
    const int c = c0 + threadIdx.x;
    if (c < C) {
      const long long orow = (long long)b * C + c;  // output row in [B*C, R]
      uint32_t out[16];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float f[32];
        float amax = 0.f;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          f[r] = __bfloat162float(tile[h * 32 + r][threadIdx.x]);
          amax = fmaxf(amax, fabsf(f[r]));
        }
        const int e = e8m0_exp(amax);
        const float inv = __int_as_float((127 - e) << 23);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
              make_float2(f[4 * q] * inv, f[4 * q + 1] * inv), __NV_SATFINITE, __NV_E4M3);
          const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
              make_float2(f[4 * q + 2] * inv, f[4 * q + 3] * inv), __NV_SATFINITE, __NV_E4M3);
          out[h * 8 + q] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        const int kb = r0 / 32 + h;
        const uint8_t sc = static_cast<uint8_t>(e + 127);
        if (sf_tiled) sf_tiled[tiled_sf_offset(static_cast<int>(orow), kb, R / 32)] = sc;
        if (sf_plain) sf_plain[orow * (R / 32) + kb] = sc;
      }
      int4* dst = reinterpret_cast<int4*>(codes + orow * R + r0);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        dst[q] = make_int4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
    }
    __syncthreads();
  }
}

}  // namespace mx
}  // namespace moe

using namespace moe;

extern "C" int moe_mxfp8_quantize(const void* x, long long ldx, int rows, int K, void* codes,
                                  long long ldc, void* sf_plain, void* sf_tiled, int w1_m,
                                  void* stream) {
  if (K % 128 || rows < 0 || (ldx % 8) || (ldc % 16) || w1_m < 0 ||
      (w1_m && (w1_m % 128 || rows % (2 * w1_m))))
    return kErrInvalidArg;
  if (rows == 0) return kOk;
  const long long n = (long long)rows * (K / 32);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long want = ceil_div_ll(n, 256);
  const int grid = static_cast<int>(want < (long long)sms * 16 ? want : (long long)sms * 16);
  mx::quant_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), ldx, rows, K, static_cast<uint8_t*>(codes), ldc,
      static_cast<uint8_t*>(sf_plain), static_cast<uint8_t*>(sf_tiled), w1_m);
  MOE_LAUNCH_CHECK();
  return kOk;
}

extern "C" int moe_mxfp8_quantize_t(const void* x, int B, int R, int C, void* codes,
                                    void* sf_tiled, void* sf_plain, void* stream) {
  if (B < 1 || R % 128 || C % 8 || ((long long)B * C) % 128) return kErrInvalidArg;
  const long long tiles = (long long)B * (R / mx::QT_ROWS) * ((C + 255) / 256);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(tiles < (long long)sms * 6 ? tiles : (long long)sms * 6);
  mx::quant_t_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), B, R, C, static_cast<uint8_t*>(codes),
      static_cast<uint8_t*>(sf_tiled), static_cast<uint8_t*>(sf_plain));
  MOE_LAUNCH_CHECK();
  return kOk;
}
