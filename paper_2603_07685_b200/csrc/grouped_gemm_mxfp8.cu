// Block-scaled MXFP8 grouped GEMM on the 5th-gen tensor cores (the
// paper's Blackwell recipe, reference emulation quant.py:166-201).
//
//   D[rows, N] = sum_k  (A_codes * 2^(sfA - 127)) (B_codes * 2^(sfB - 127))^T,  fp32 in TMEM
//
// A: E4M3 codes [rows, K] (the padded expert-major plan), B: E4M3 codes [E * N, K] (K-major
// expert weights), both with 1x32-block E8M0 scales in the tiled layout written by
// moe_mxfp8_quantize / the fc1 epilogue. tcgen05.mma.kind::mxf8f6f4.block_scale, UMMA
// 128 x 128 x 32, one CTA per SM (persistent), warp-specialised like the bf16 engine:
//   warp 0: TMA (A, B tiles; scale chunks by 1-D bulk copies), warp 1: tcgen05.cp of the
//   scale chunks smem -> TMEM, then 4 block-scaled MMAs per 128-wide K stage, warps 2-5:
//   epilogue from a double-buffered TMEM accumulator.
// TMEM: accumulators at columns [0, 256), scale factors at [256, 264) (SFA 4 columns, SFB 4
// columns: row r's scale for the stage's K-block j is byte j of column r / 32, lane r % 32,
// replicated over the 4 lane quarters by tcgen05.cp 32x128b.warpx4).
//
// Epilogues: EPI_BF16 (fc2: bf16 rows) and EPI_SWIGLU_Q (fc1: the MXFP8 W1 copy interleaves
// gate/up in 64-row blocks, so every 128-wide tile holds matching gate and up columns; it
// writes preact in the bf16 engine's 128-interleaved layout, act in bf16, AND act quantised
// to MXFP8 -- each thread holds exactly one 32-element block of its row -- so fc2 reads
// fp8 codes without a separate quantisation pass).
#include <cudaTypedefs.h>
#include <cuda_fp8.h>

#include <mutex>

#include "common.cuh"

namespace moe {
namespace mx8 {

constexpr int BM = 128, BK = 128;  // BK in fp8 elements (= bytes)
constexpr int UMMA_K = 32;
constexpr int A_STAGE = BM * BK, SF_CHUNK = 512;
// CG = 1: UMMA 128 x 128 per CTA. CG = 2: CTA pair, UMMA 256 x 128 (cta_group::2): each CTA
// stages its 128 rows of A and half (64 rows) of the B tile, and its own copy of both scale
// chunks; per-SM shared-memory operand traffic drops from 8 KB to 6 KB per 1 MFLOP and the
// ring holds 8 stages instead of 6 (more time to hide TMA latency at fp8 MMA rates).
// WIDE: 256-wide N tiles with a single TMEM accumulator (256 columns + 12 scale columns);
// the operand traffic per MMA FLOP drops by a third again, at the cost of an epilogue that
// no longer overlaps the next tile's MMAs. Narrow: 128-wide tiles, double-buffered.
template <int CG, bool WIDE>
struct Cfg {
  static constexpr int BN = WIDE ? 256 : 128;
  static constexpr int ACC = WIDE ? 1 : 2;        // accumulator stages in TMEM
  static constexpr int SFB_CHUNKS = BN / 128;
  static constexpr int B_ROWS = BN / CG;
  static constexpr int B_STAGE = B_ROWS * BK;
  static constexpr int STAGE = A_STAGE + B_STAGE + (1 + SFB_CHUNKS) * SF_CHUNK;
  static constexpr int FIT = 200704 / STAGE;
  static constexpr int STAGES = FIT > 8 ? 8 : FIT;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};
constexpr int TMEM_COLS = 512;
constexpr int SF_COL = 256;
// epilogue warps: 4 (one per TMEM lane quarter), 8 for the single-accumulator wide tiles
// (two per quarter, each draining half the columns: the MMAs wait for the drain there)
template <bool WIDE>
constexpr int epi_warps() { return WIDE ? 8 : 4; }
constexpr int BAND_M = 16;

enum Epi : int { EPI_BF16 = 0, EPI_SWIGLU_Q = 1, EPI_DSWIGLU_Q = 2 };

__device__ __forceinline__ int e8m0_exp(float amax) {
  if (!(amax > 0.f)) return -127;
  int q;
  const float f = frexpf(amax, &q);
  int e = q - 9 + (f > 0.875f ? 1 : 0);
  return e < -127 ? -127 : (e > 127 ? 127 : e);
}


struct Params {
  const int* num_m_blocks;
  const int* block_expert;
  int N, K;
  const uint8_t* sfa;  // tiled, per (128-row tile, K stage) 512 B
  const uint8_t* sfb;
  void* out;           // EPI_BF16: bf16 [rows, ldo]; EPI_SWIGLU_Q: preact [rows, 2m]
  long long ldo;
  void* act;           // EPI_SWIGLU_Q: bf16 [rows, m] (nullable)
  uint8_t* act_q;      // EPI_SWIGLU_Q: E4M3 codes [rows, m]
  uint8_t* act_sf;     // EPI_SWIGLU_Q: tiled scales for K = m
  int m;
  // EPI_DSWIGLU_Q (fc2 dgrad): out = d_preact [rows, 2m] (interleaved like preact),
  // aux = preact, act_q / act_sf = d_preact quantised along 2m (fc1 dgrad's A operand)
  const __nv_bfloat16* aux;
  int num_experts_gk;
  // grouped-K (weight gradients): expert e reduces K rows [k_off[e], k_off[e+1]) of the
  // transposed operands A^T [M, K], B^T [N, K]; out[e] = M x N at out + e * out_stride
  const int* k_off;
  int M;
  long long out_stride;
  // transposed MXFP8 copy of the epilogue's activation (EPI_SWIGLU_Q: act, EPI_DSWIGLU_Q:
  // d_preact), quantised along the token rows for the weight-gradient GEMM: codes [C, ldT]
  // (C = m or 2m columns become rows), tiled scales; nullable
  uint8_t* qt;
  uint8_t* qt_sf;
  long long qt_ld;
};

// Column-wise (token-row) quantisation from registers: the 32 lanes of a warp hold 32
// consecutive rows (TMEM lanes), lane l has v[j] = value of (row0 + l, col0 + j). For each
// column, a 5-step butterfly gives the block amax over the 32 rows; each lane then writes its
// code byte (the 32 lanes write 32 contiguous bytes of output row col0 + j).
__device__ __forceinline__ void quant_t_cols(const float (&v)[32], int col0, long long row0,
                                             uint8_t* qt, uint8_t* qt_sf, long long ldT) {
  const int lane = threadIdx.x & 31;
  const int kblocks = static_cast<int>(ldT / 32);
  const int kb = static_cast<int>(row0 / 32);
#pragma unroll 4
  for (int j = 0; j < 32; ++j) {
    float a = fabsf(v[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    const int e = e8m0_exp(a);
    const float inv = __int_as_float((127 - e) << 23);
    const __nv_fp8x2_storage_t c2 =
        __nv_cvt_float2_to_fp8x2(make_float2(v[j] * inv, 0.f), __NV_SATFINITE, __NV_E4M3);
    const long long orow = col0 + j;
    qt[orow * ldT + row0 + lane] = static_cast<uint8_t>(c2 & 0xFF);
    if (lane == 0) {
      const int r = static_cast<int>(orow);
      qt_sf[((long long)(r >> 7) * (kblocks >> 2) + (kb >> 2)) * 512 + (r & 31) * 16 +
            ((r & 127) >> 5) * 4 + (kb & 3)] = static_cast<uint8_t>(e + 127);
    }
  }
}

// E4M3-quantise 32 values (one MX block), write 32 codes + the scale byte (tiled layout).
__device__ __forceinline__ void quant_block32(const float (&v)[32], uint8_t* codes_dst,
                                              uint8_t* sf, long long row, int kb,
                                              int kblocks) {
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) amax = fmaxf(amax, fabsf(v[i]));
  const int e = e8m0_exp(amax);
  const float inv = __int_as_float((127 - e) << 23);
  uint32_t qv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
        make_float2(v[4 * k] * inv, v[4 * k + 1] * inv), __NV_SATFINITE, __NV_E4M3);
    const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
        make_float2(v[4 * k + 2] * inv, v[4 * k + 3] * inv), __NV_SATFINITE, __NV_E4M3);
    qv[k] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
  }
  int4* qd = reinterpret_cast<int4*>(codes_dst);
  qd[0] = make_int4(qv[0], qv[1], qv[2], qv[3]);
  qd[1] = make_int4(qv[4], qv[5], qv[6], qv[7]);
  const int rr = static_cast<int>(row & 127);
  sf[((row >> 7) * (kblocks >> 2) + (kb >> 2)) * 512 + (rr & 31) * 16 + (rr >> 5) * 4 +
     (kb & 3)] = static_cast<uint8_t>(e + 127);
}

// 32 rows x 16 B, no swizzle, rows contiguous (core matrices 8 x 16 B, SBO 128 B)
__device__ __forceinline__ uint64_t sf_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((128u >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((128u >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;  // layout type 0: SWIZZLE_NONE
}
__device__ __forceinline__ void tmem_cp_sf(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc)
               : "memory");
}
// Block-scaled instruction descriptor: E4M3 x E4M3, E8M0 scales, K-major, M=128, N=128.
__host__ __device__ constexpr uint32_t idesc_mx(int j, int M, int N) {
  return (static_cast<uint32_t>(j) << 4)          // B scale-factor id (byte)
         | (0u << 7) | (0u << 10)                 // A, B format: E4M3
         | (static_cast<uint32_t>(N >> 3) << 17)   // N / 8
         | (1u << 23)                             // scale format: E8M0
         | (static_cast<uint32_t>(M >> 4) << 24)   // M / 16
         | (static_cast<uint32_t>(j) << 29);      // A scale-factor id
}
__device__ __forceinline__ void umma_mx_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_cp_sf_pair(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc)
               : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const void* tmap,
                                                 uint64_t* bar, int x, int y) {
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_leader), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_mx(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + __expf(-g)); }


struct Tile {
  int expert, m0, n0, k0, nkb;
};
template <int CG, int BN, bool GK>
__device__ __forceinline__ void decode_tile(const Params& p, int t, int num_units, int rank,
                                            Tile& tl) {
  const int nb_count = p.N / BN;
  if constexpr (GK) {
    const int per_e = (p.M / (BM * CG)) * nb_count;
    const int e = t / per_e, rem = t - e * per_e;
    const int mu = rem / nb_count, nb = rem - mu * nb_count;
    tl.expert = e;
    tl.m0 = mu * BM * CG + rank * BM;
    tl.n0 = nb * BN;
    tl.k0 = __ldg(p.k_off + e);
    tl.nkb = (__ldg(p.k_off + e + 1) - tl.k0) / BK;
    return;
  }
  tl.k0 = 0;
  tl.nkb = p.K / BK;
  const int band = t / (BAND_M * nb_count);
  const int rem = t - band * BAND_M * nb_count;
  const int u0 = band * BAND_M;
  const int rows = min(BAND_M, num_units - u0);
  const int nb = rem / rows;
  const int u = u0 + (rem - nb * rows);
  tl.expert = __ldg(p.block_expert + u * CG);
  tl.m0 = u * BM * CG + rank * BM;
  tl.n0 = nb * BN;
}

template <int EPI, int CG, bool WIDE, bool GK>
__global__ void __launch_bounds__(64 + 32 * epi_warps<WIDE>(), 1)
    mxfp8_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                      const __grid_constant__ CUtensorMap tmap_b,
                      const __grid_constant__ CUtensorMap tmap_sfa,
                      const __grid_constant__ CUtensorMap tmap_sfb, const Params p) {
  using C = Cfg<CG, WIDE>;
  constexpr int BN = C::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  auto sa = [&](int s) { return smem + s * C::STAGE; };
  auto sb = [&](int s) { return smem + s * C::STAGE + A_STAGE; };
  auto ssfa = [&](int s) { return smem + s * C::STAGE + A_STAGE + C::B_STAGE; };
  auto ssfb = [&](int s) { return smem + s * C::STAGE + A_STAGE + C::B_STAGE + SF_CHUNK; };

  const int warp = warp_id(), lane = lane_id();
  const int rank = CG == 2 ? static_cast<int>(cluster_rank()) : 0;
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    tma_prefetch_desc(&tmap_sfa);
    tma_prefetch_desc(&tmap_sfb);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < C::ACC; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], epi_warps<WIDE>() * CG);
    }
    fence_mbar_init();
    fence_async_shared();
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      tmem_alloc<TMEM_COLS>(tmem_slot);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync_all();
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_units = GK ? 0 : *p.num_m_blocks / CG;
  const int num_tiles = GK ? p.num_experts_gk * (p.M / (BM * CG)) * (p.N / BN)
                           : num_units * (p.N / BN);
  const int kst = p.K / BK;  // K stages per 128-row scale tile
  const int first = blockIdx.x / CG, stride = gridDim.x / CG;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = first; t < num_tiles; t += stride) {
        Tile tl;
        decode_tile<CG, BN, GK>(p, t, num_units, rank, tl);
        // first B row of the (full) N tile: stacked weights [E*N, K], or B^T [N, K] (GK)
        const int brow = GK ? tl.n0 : tl.expert * p.N + tl.n0;
        for (int kq = 0; kq < tl.nkb; ++kq) {
          const int kb = tl.k0 / BK + kq;  // global K stage
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full_bar[s], C::STAGE * CG);
          auto load = [&](void* dst, const CUtensorMap* tm, int x, int y) {
            if constexpr (CG == 1)
              tma_load_2d(dst, tm, &full_bar[s], x, y);
            else
              tma_load_2d_pair(dst, tm, &full_bar[s], x, y);
          };
          load(sa(s), &tmap_a, kb * BK, tl.m0);
          load(sb(s), &tmap_b, kb * BK, brow + rank * C::B_ROWS);
          // scale chunks viewed as [chunks * 2, 256] bytes: box {256, 2} = one 512-B chunk;
          // each CTA holds the chunk of its own 128 A rows and the full N tile's B chunk
          load(ssfa(s), &tmap_sfa, 0, ((tl.m0 / BM) * kst + kb) * 2);
#pragma unroll
          for (int c = 0; c < C::SFB_CHUNKS; ++c)
            load(ssfb(s) + c * SF_CHUNK, &tmap_sfb, 0, ((brow / 128 + c) * kst + kb) * 2);
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      const uint32_t t_sfa = tmem_base + SF_COL, t_sfb = tmem_base + SF_COL + 4;
      for (int t = first; t < num_tiles; t += stride) {
        int nkb = p.K / BK;
        if constexpr (GK) {
          Tile tl;
          decode_tile<CG, BN, GK>(p, t, num_units, rank, tl);
          nkb = tl.nkb;
          if (nkb == 0) continue;  // expert without rows: the epilogue writes zeros
        }
        mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          // scale chunks smem -> TMEM (ordered before the MMAs below: same tcgen05 pipe;
          // with cta_group::2 each CTA's chunk goes to its own TMEM)
          if constexpr (CG == 1) {
            tmem_cp_sf(t_sfa, sf_desc(smem_u32(ssfa(s))));
#pragma unroll
            for (int c = 0; c < C::SFB_CHUNKS; ++c)
              tmem_cp_sf(t_sfb + 4 * c, sf_desc(smem_u32(ssfb(s) + c * SF_CHUNK)));
          } else {
            tmem_cp_sf_pair(t_sfa, sf_desc(smem_u32(ssfa(s))));
#pragma unroll
            for (int c = 0; c < C::SFB_CHUNKS; ++c)
              tmem_cp_sf_pair(t_sfb + 4 * c, sf_desc(smem_u32(ssfb(s) + c * SF_CHUNK)));
          }
          const uint32_t a_base = smem_u32(sa(s)), b_base = smem_u32(sb(s));
#pragma unroll
          for (int j = 0; j < BK / UMMA_K; ++j) {
            const uint64_t ad = make_sdesc_sw128(a_base + j * UMMA_K, 16, 1024);
            const uint64_t bd = make_sdesc_sw128(b_base + j * UMMA_K, 16, 1024);
            if constexpr (CG == 1)
              umma_mx(d_tmem, ad, bd, idesc_mx(j, BM, BN), t_sfa, t_sfb,
                      (kb | j) != 0 ? 1u : 0u);
            else
              umma_mx_pair(d_tmem, ad, bd, idesc_mx(j, 2 * BM, BN), t_sfa, t_sfb,
                           (kb | j) != 0 ? 1u : 0u);
          }
          if constexpr (CG == 1)
            umma_commit(&empty_bar[s]);
          else
            umma_commit_pair(&empty_bar[s]);
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if constexpr (CG == 1)
          umma_commit(&tfull_bar[acc]);
        else
          umma_commit_pair(&tfull_bar[acc]);
        if (++acc == C::ACC) {
          acc = 0;
          acc_ph ^= 1;
        }
      }
    }
  } else {
    constexpr int NPART = epi_warps<WIDE>() / 4;  // warps sharing a lane quarter
    const int part = (warp - 2) / 4;
    const int q = warp & 3;
    const int row_local = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = first; t < num_tiles; t += stride) {
      Tile tl;
      decode_tile<CG, BN, GK>(p, t, num_units, rank, tl);
      const long long row = tl.m0 + row_local;
      if constexpr (GK) {
        if (tl.nkb == 0) {  // weight gradient of an expert without rows: exactly zero
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) +
                             tl.expert * p.out_stride + row * p.ldo + tl.n0;
          for (int c = part * (BN / 8 / NPART); c < (part + 1) * (BN / 8 / NPART); ++c)
            reinterpret_cast<int4*>(o)[c] = make_int4(0, 0, 0, 0);
          continue;
        }
      }
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
      const uint32_t t_base = tmem_base + lane_off + acc * BN;
      if constexpr (EPI == EPI_BF16) {
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) +
                           (GK ? tl.expert * p.out_stride : 0) + row * p.ldo + tl.n0;
#pragma unroll 1
        for (int c = part * (BN / 32 / NPART); c < (part + 1) * (BN / 32 / NPART); ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_base + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            int4 w;
            w.x = pack_bf16x2(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1]));
            w.y = pack_bf16x2(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3]));
            w.z = pack_bf16x2(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5]));
            w.w = pack_bf16x2(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7]));
            reinterpret_cast<int4*>(o + c * 32)[v] = w;
          }
        }
      } else if constexpr (EPI == EPI_DSWIGLU_Q) {
        // accumulator = dL/d(act) for activation columns [n0, n0 + BN); recompute the SwiGLU
        // derivative from the saved pre-activation (interleaved gate/up, 128-column blocks)
        const __nv_bfloat16* pre_row = p.aux + row * (2LL * p.m);
        __nv_bfloat16* dpre_row = reinterpret_cast<__nv_bfloat16*>(p.out) + row * (2LL * p.m);
        const int kblocks = 2 * p.m / 32;
#pragma unroll 1
        for (int c = part * (BN / 32 / NPART); c < (part + 1) * (BN / 32 / NPART); ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_base + c * 32, r);
          const int j0 = tl.n0 + c * 32;
          const long long pos = (long long)(j0 >> 7) * 256 + (j0 & 127);
          int4 gv[4], uv[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            gv[v] = reinterpret_cast<const int4*>(pre_row + pos)[v];
            uv[v] = reinterpret_cast<const int4*>(pre_row + pos + 128)[v];
          }
          tmem_ld_wait();
          float dg[32], du[32];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const uint32_t* sg = reinterpret_cast<const uint32_t*>(&gv[v]);
            const uint32_t* su = reinterpret_cast<const uint32_t*>(&uv[v]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 gg = unpack_bf16x2(sg[j]);
              const float2 uu = unpack_bf16x2(su[j]);
              const int i = 8 * v + 2 * j;
              const float a0 = __uint_as_float(r[i]), a1 = __uint_as_float(r[i + 1]);
              const float s0 = 1.0f / (1.0f + __expf(-gg.x));
              const float s1 = 1.0f / (1.0f + __expf(-gg.y));
              dg[i] = a0 * uu.x * s0 * (1.0f + gg.x * (1.0f - s0));
              dg[i + 1] = a1 * uu.y * s1 * (1.0f + gg.y * (1.0f - s1));
              du[i] = a0 * gg.x * s0;
              du[i + 1] = a1 * gg.y * s1;
            }
          }
          // bf16 d_preact (the wgrad operand), then quantise the bf16 values
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            int4 wg, wu;
            uint32_t* pg = reinterpret_cast<uint32_t*>(&wg);
            uint32_t* pu = reinterpret_cast<uint32_t*>(&wu);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = 8 * v + 2 * j;
              pg[j] = pack_bf16x2(dg[i], dg[i + 1]);
              pu[j] = pack_bf16x2(du[i], du[i + 1]);
              const float2 bg = unpack_bf16x2(pg[j]), bu = unpack_bf16x2(pu[j]);
              dg[i] = bg.x;
              dg[i + 1] = bg.y;
              du[i] = bu.x;
              du[i + 1] = bu.y;
            }
            reinterpret_cast<int4*>(dpre_row + pos)[v] = wg;
            reinterpret_cast<int4*>(dpre_row + pos + 128)[v] = wu;
          }
          if (p.qt) {
            quant_t_cols(dg, static_cast<int>(pos), tl.m0 + q * 32, p.qt, p.qt_sf, p.qt_ld);
            quant_t_cols(du, static_cast<int>(pos + 128), tl.m0 + q * 32, p.qt, p.qt_sf,
                         p.qt_ld);
          }
          quant_block32(dg, p.act_q + row * (2LL * p.m) + pos, p.act_sf, row,
                        static_cast<int>(pos / 32), kblocks);
          quant_block32(du, p.act_q + row * (2LL * p.m) + pos + 128, p.act_sf, row,
                        static_cast<int>((pos + 128) / 32), kblocks);
        }
      } else {
        // tile columns [0, BN/2) = gate rows g0 + [0, BN/2), [BN/2, BN) = the matching up
        // rows (narrow tiles: W1 in 64-row gate/up blocks; wide: the bf16 engine's 128)
        constexpr int HALF = BN / 2;
        const int g0 = tl.n0 / 2;
        __nv_bfloat16* pre = reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.ldo +
                             (g0 >> 7) * 256 + (g0 & 127);
#pragma unroll 1
        for (int c = part * (HALF / 32 / NPART); c < (part + 1) * (HALF / 32 / NPART); ++c) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(t_base + c * 32, g);
          tmem_ld_32x32b_x32(t_base + HALF + c * 32, u);
          tmem_ld_wait();
          uint32_t a2[16];
          float amax = 0.f;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float g_0 = __uint_as_float(g[2 * i]), g_1 = __uint_as_float(g[2 * i + 1]);
            const float u_0 = __uint_as_float(u[2 * i]), u_1 = __uint_as_float(u[2 * i + 1]);
            a2[i] = pack_bf16x2(silu_f(g_0) * u_0, silu_f(g_1) * u_1);
            const float2 ab = unpack_bf16x2(a2[i]);  // quantise the bf16 activation
            amax = fmaxf(amax, fmaxf(fabsf(ab.x), fabsf(ab.y)));
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            int4 wg, wu;
            uint32_t* pg = reinterpret_cast<uint32_t*>(&wg);
            uint32_t* pu = reinterpret_cast<uint32_t*>(&wu);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = 8 * v + 2 * j;
              pg[j] = pack_bf16x2(__uint_as_float(g[i]), __uint_as_float(g[i + 1]));
              pu[j] = pack_bf16x2(__uint_as_float(u[i]), __uint_as_float(u[i + 1]));
            }
            reinterpret_cast<int4*>(pre + c * 32)[v] = wg;
            reinterpret_cast<int4*>(pre + 128 + c * 32)[v] = wu;
          }
          const int col = g0 + c * 32;  // activation column = MX block col / 32
          if (p.qt) {
            float vt[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 ab = unpack_bf16x2(a2[i]);
              vt[2 * i] = ab.x;
              vt[2 * i + 1] = ab.y;
            }
            quant_t_cols(vt, col, tl.m0 + q * 32, p.qt, p.qt_sf, p.qt_ld);
          }
          if (p.act) {
            int4* ad = reinterpret_cast<int4*>(reinterpret_cast<__nv_bfloat16*>(p.act) +
                                               row * p.m + col);
#pragma unroll
            for (int v = 0; v < 4; ++v)
              ad[v] = make_int4(a2[4 * v], a2[4 * v + 1], a2[4 * v + 2], a2[4 * v + 3]);
          }
          const int e = e8m0_exp(amax);
          const float inv = __int_as_float((127 - e) << 23);
          uint32_t qv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float2 x0 = unpack_bf16x2(a2[2 * k]), x1 = unpack_bf16x2(a2[2 * k + 1]);
            const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
                make_float2(x0.x * inv, x0.y * inv), __NV_SATFINITE, __NV_E4M3);
            const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
                make_float2(x1.x * inv, x1.y * inv), __NV_SATFINITE, __NV_E4M3);
            qv[k] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
          }
          int4* qd = reinterpret_cast<int4*>(p.act_q + row * p.m + col);
          qd[0] = make_int4(qv[0], qv[1], qv[2], qv[3]);
          qd[1] = make_int4(qv[4], qv[5], qv[6], qv[7]);
          const int kb = col / 32, kblocks = p.m / 32;
          const int rr = static_cast<int>(row & 127);
          p.act_sf[((row >> 7) * (kblocks >> 2) + (kb >> 2)) * 512 + (rr & 31) * 16 +
                   (rr >> 5) * 4 + (kb & 3)] = static_cast<uint8_t>(e + 127);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1)
          mbar_arrive(&tempty_bar[acc]);
        else
          mbar_arrive_leader(&tempty_bar[acc]);
      }
      if (++acc == C::ACC) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync_all();
  } else {
    __syncthreads();
  }
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 1) {
      tmem_dealloc<TMEM_COLS>(tmem_base);
    } else {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(TMEM_COLS)
                   : "memory");
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}
// 2-D u8 tensor [outer, inner] with box {box_inner, box_outer}
static int make_tmap_u8(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                        uint32_t box_inner, uint32_t box_outer, bool swizzle) {
  auto fn = encode_fn();
  if (!fn) return kErrCuda;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (inner & 15)) return kErrInvalidArg;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? kOk : kErrCuda;
}

template <int EPI, int CG, bool WIDE, bool GK>
static int launch_cg(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tsa,
                     const CUtensorMap& tsb, const Params& p, int max_m_blocks,
                     cudaStream_t stream) {
  using C = Cfg<CG, WIDE>;
  auto kern = mxfp8_gemm_kernel<EPI, CG, WIDE, GK>;
  MOE_CUDA_CHECK(ensure_dyn_smem(reinterpret_cast<const void*>(kern), C::SMEM));
  const int sms = device_sms();
  const int tiles = GK ? p.num_experts_gk * (p.M / (BM * CG)) * (p.N / C::BN)
                     : (max_m_blocks / CG) * (p.N / C::BN);
  if (tiles <= 0) return kOk;
  int grid = tiles * CG < sms ? tiles * CG : sms;
  grid -= grid % CG;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64 + 32 * epi_warps<WIDE>());
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MOE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ta, tb, tsa, tsb, p));
  return kOk;
}

template <int EPI>
static int launch(const void* a, int a_rows, int max_rows, const void* b, int num_experts,
                  Params p, int pair, int wide, cudaStream_t stream) {
  CUtensorMap ta, tb, tsa, tsb;
  int st;
  const int cg = pair ? 2 : 1;
  const int bn = wide ? 256 : 128;
  const long long b_rows = (long long)num_experts * p.N;
  if ((st = make_tmap_u8(&ta, a, p.K, a_rows, BK, BM, true))) return st;
  if ((st = make_tmap_u8(&tb, b, p.K, b_rows, BK, bn / cg, true))) return st;
  // scale chunks: [rows/128 * K/128 chunks] x 512 B viewed as [2 * chunks, 256]
  const long long sfa_chunks = (long long)(max_rows / BM) * (p.K / BK);
  const long long sfb_chunks = (b_rows / 128) * (p.K / BK);
  if ((st = make_tmap_u8(&tsa, p.sfa, 256, 2 * sfa_chunks, 256, 2, false))) return st;
  if ((st = make_tmap_u8(&tsb, p.sfb, 256, 2 * sfb_chunks, 256, 2, false))) return st;
  const int mb = max_rows / BM;
  if (pair)
    return wide ? launch_cg<EPI, 2, true, false>(ta, tb, tsa, tsb, p, mb, stream)
                : launch_cg<EPI, 2, false, false>(ta, tb, tsa, tsb, p, mb, stream);
  return wide ? launch_cg<EPI, 1, true, false>(ta, tb, tsa, tsb, p, mb, stream)
              : launch_cg<EPI, 1, false, false>(ta, tb, tsa, tsb, p, mb, stream);
}

// grouped-K weight gradient: A^T codes [M, K], B^T codes [N, K], K = token rows
static int launch_wgrad(const void* at, const void* bt, Params p, int pair, int wide,
                        cudaStream_t stream) {
  CUtensorMap ta, tb, tsa, tsb;
  int st;
  const int cg = pair ? 2 : 1;
  const int bn = wide ? 256 : 128;
  if ((st = make_tmap_u8(&ta, at, p.K, p.M, BK, BM, true))) return st;
  if ((st = make_tmap_u8(&tb, bt, p.K, p.N, BK, bn / cg, true))) return st;
  const long long sfa_chunks = (long long)(p.M / BM) * (p.K / BK);
  const long long sfb_chunks = (long long)(p.N / 128) * (p.K / BK);
  if ((st = make_tmap_u8(&tsa, p.sfa, 256, 2 * sfa_chunks, 256, 2, false))) return st;
  if ((st = make_tmap_u8(&tsb, p.sfb, 256, 2 * sfb_chunks, 256, 2, false))) return st;
  if (pair)
    return wide ? launch_cg<EPI_BF16, 2, true, true>(ta, tb, tsa, tsb, p, 0, stream)
                : launch_cg<EPI_BF16, 2, false, true>(ta, tb, tsa, tsb, p, 0, stream);
  return wide ? launch_cg<EPI_BF16, 1, true, true>(ta, tb, tsa, tsb, p, 0, stream)
              : launch_cg<EPI_BF16, 1, false, true>(ta, tb, tsa, tsb, p, 0, stream);
}

}  // namespace mx8
}  // namespace moe

using namespace moe;
using namespace moe::mx8;

extern "C" {

// out[rows, N] (bf16) = A x B_e^T with MXFP8 operands (fc2 forward: A = act codes [rows, m],
// B = W2 codes [E, h, m]).
int moe_gg_mxfp8_gemm(const void* a, const void* sfa, int a_rows, int max_rows, int K, int N,
                      const void* b, const void* sfb, int num_experts, const int* block_expert,
                      const int* num_m_blocks, void* out, int flags, void* stream) {
  const int pair = flags & 1, wide = (flags >> 1) & 1;
  if (K % BK || N % (wide ? 256 : 128) || max_rows % (BM * (pair ? 2 : 1)) || a_rows > max_rows)
    return kErrInvalidArg;
  Params p{};
  p.num_m_blocks = num_m_blocks;
  p.block_expert = block_expert;
  p.N = N;
  p.K = K;
  p.sfa = static_cast<const uint8_t*>(sfa);
  p.sfb = static_cast<const uint8_t*>(sfb);
  p.out = out;
  p.ldo = N;
  return launch<EPI_BF16>(a, a_rows, max_rows, b, num_experts, p, pair, wide,
                          static_cast<cudaStream_t>(stream));
}

// fc1 forward + SwiGLU with MXFP8 operands: B = W1 codes [E, 2m, h] interleaved gate/up in
// 64-row blocks (moe_mxfp8_interleave_w1). Writes preact (bf16, the bf16 engine's
// 128-interleaved layout), act (bf16, nullable) and act as MXFP8 (codes + tiled scales).
static int mxfp8_fc1_impl(const void* xq, const void* sfx, int a_rows, int max_rows, int h,
                          int m, const void* w1q, const void* sfw, int num_experts,
                          const int* block_expert, const int* num_m_blocks, void* preact,
                          void* act, void* act_q, void* act_sf, void* act_t, void* act_t_sf,
                          int flags, void* stream);

int moe_gg_mxfp8_fc1(const void* xq, const void* sfx, int a_rows, int max_rows, int h, int m,
                     const void* w1q, const void* sfw, int num_experts, const int* block_expert,
                     const int* num_m_blocks, void* preact, void* act, void* act_q,
                     void* act_sf, int flags, void* stream) {
  return mxfp8_fc1_impl(xq, sfx, a_rows, max_rows, h, m, w1q, sfw, num_experts, block_expert,
                        num_m_blocks, preact, act, act_q, act_sf, nullptr, nullptr, flags,
                        stream);
}

// ... and act quantised along the token rows too (act_t: codes [m, max_rows], tiled scales):
// the weight-gradient GEMM's operand straight from the epilogue (warp-shuffle block amax).
int moe_gg_mxfp8_fc1_t(const void* xq, const void* sfx, int a_rows, int max_rows, int h, int m,
                       const void* w1q, const void* sfw, int num_experts,
                       const int* block_expert, const int* num_m_blocks, void* preact,
                       void* act, void* act_q, void* act_sf, void* act_t, void* act_t_sf,
                       int flags, void* stream) {
  if (!act_t || !act_t_sf) return kErrInvalidArg;
  return mxfp8_fc1_impl(xq, sfx, a_rows, max_rows, h, m, w1q, sfw, num_experts, block_expert,
                        num_m_blocks, preact, act, act_q, act_sf, act_t, act_t_sf, flags,
                        stream);
}

static int mxfp8_fc1_impl(const void* xq, const void* sfx, int a_rows, int max_rows, int h,
                          int m, const void* w1q, const void* sfw, int num_experts,
                          const int* block_expert, const int* num_m_blocks, void* preact,
                          void* act, void* act_q, void* act_sf, void* act_t, void* act_t_sf,
                          int flags, void* stream) {
  const int pair = flags & 1, wide = (flags >> 1) & 1;
  if (h % BK || m % 128 || max_rows % (BM * (pair ? 2 : 1)) || a_rows > max_rows || !act_q ||
      !act_sf)
    return kErrInvalidArg;
  Params p{};
  p.num_m_blocks = num_m_blocks;
  p.block_expert = block_expert;
  p.N = 2 * m;
  p.K = h;
  p.sfa = static_cast<const uint8_t*>(sfx);
  p.sfb = static_cast<const uint8_t*>(sfw);
  p.out = preact;
  p.ldo = 2 * m;
  p.act = act;
  p.act_q = static_cast<uint8_t*>(act_q);
  p.act_sf = static_cast<uint8_t*>(act_sf);
  p.m = m;
  p.qt = static_cast<uint8_t*>(act_t);
  p.qt_sf = static_cast<uint8_t*>(act_t_sf);
  p.qt_ld = max_rows;
  return launch<EPI_SWIGLU_Q>(xq, a_rows, max_rows, w1q, num_experts, p, pair, wide,
                              static_cast<cudaStream_t>(stream));
}

}  // extern "C"

extern "C" {

// fc2 data-gradient fused with the SwiGLU backward, MXFP8 operands: A = dO codes [rows, h]
// (1x32 along h), B = W2^T codes [E*m, h] (moe_mxfp8_quantize_t of W2 [E, h, m]). Writes
// d_preact (bf16, preact's interleaved layout; the wgrad operand) and d_preact quantised
// along 2m (codes + tiled scales: fc1 dgrad's A operand). Standard combine (no row scale).
int moe_gg_mxfp8_fc2_dgrad_t(const void* doq, const void* sfd, int a_rows, int max_rows,
                             int h, int m, const void* w2tq, const void* sfw, int num_experts,
                             const int* block_expert, const int* num_m_blocks,
                             const void* preact, void* d_preact, void* dpre_q, void* dpre_sf,
                             void* dpre_t, void* dpre_t_sf, int flags, void* stream);

int moe_gg_mxfp8_fc2_dgrad(const void* doq, const void* sfd, int a_rows, int max_rows, int h,
                           int m, const void* w2tq, const void* sfw, int num_experts,
                           const int* block_expert, const int* num_m_blocks, const void* preact,
                           void* d_preact, void* dpre_q, void* dpre_sf, int flags,
                           void* stream) {
  return moe_gg_mxfp8_fc2_dgrad_t(doq, sfd, a_rows, max_rows, h, m, w2tq, sfw, num_experts,
                                  block_expert, num_m_blocks, preact, d_preact, dpre_q,
                                  dpre_sf, nullptr, nullptr, flags, stream);
}

// ... and d_preact quantised along the token rows too (dpre_t: codes [2m, max_rows]).
int moe_gg_mxfp8_fc2_dgrad_t(const void* doq, const void* sfd, int a_rows, int max_rows,
                             int h, int m, const void* w2tq, const void* sfw, int num_experts,
                             const int* block_expert, const int* num_m_blocks,
                             const void* preact, void* d_preact, void* dpre_q, void* dpre_sf,
                             void* dpre_t, void* dpre_t_sf, int flags, void* stream) {
  const int pair = flags & 1, wide = (flags >> 1) & 1;
  if (h % BK || m % (wide ? 256 : 128) || max_rows % (BM * (pair ? 2 : 1)) ||
      a_rows > max_rows || !dpre_q || !dpre_sf || !preact)
    return kErrInvalidArg;
  Params p{};
  p.num_m_blocks = num_m_blocks;
  p.block_expert = block_expert;
  p.N = m;
  p.K = h;
  p.sfa = static_cast<const uint8_t*>(sfd);
  p.sfb = static_cast<const uint8_t*>(sfw);
  p.out = d_preact;
  p.ldo = 2 * m;
  p.aux = static_cast<const __nv_bfloat16*>(preact);
  p.act_q = static_cast<uint8_t*>(dpre_q);
  p.act_sf = static_cast<uint8_t*>(dpre_sf);
  p.m = m;
  p.qt = static_cast<uint8_t*>(dpre_t);
  p.qt_sf = static_cast<uint8_t*>(dpre_t_sf);
  p.qt_ld = max_rows;
  return launch<EPI_DSWIGLU_Q>(doq, a_rows, max_rows, w2tq, num_experts, p, pair, wide,
                               static_cast<cudaStream_t>(stream));
}

}  // extern "C"

extern "C" {

// Weight gradient on MXFP8 operands: dw[e] (bf16 [M, N]) = sum over token rows
// [k_off[e], k_off[e+1]) of A[r, 0:M]^T B[r, 0:N], with A^T / B^T given as codes [M, K] /
// [N, K] quantised along the token rows (moe_mxfp8_quantize_t of the [K, M] / [K, N]
// activations). k_off[] are multiples of 128 (the padded plan; padding rows are zero).
int moe_gg_mxfp8_wgrad(const void* at, const void* sfa, const void* bt, const void* sfb, int K,
                       int M, int N, int num_experts, const int* k_off, void* dw, int flags,
                       void* stream) {
  const int pair = flags & 1, wide = (flags >> 1) & 1;
  if (K % BK || M % (BM * (pair ? 2 : 1)) || N % (wide ? 256 : 128) || !k_off)
    return kErrInvalidArg;
  Params p{};
  p.N = N;
  p.K = K;
  p.M = M;
  p.sfa = static_cast<const uint8_t*>(sfa);
  p.sfb = static_cast<const uint8_t*>(sfb);
  p.out = dw;
  p.ldo = N;
  p.out_stride = (long long)M * N;
  p.k_off = k_off;
  p.num_experts_gk = num_experts;
  return launch_wgrad(at, bt, p, pair, wide, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
