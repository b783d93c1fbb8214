// Grouped GEMM for the MoE expert FFN on sm_100a: tcgen05.mma (bf16 in, fp32 in TMEM),
// TMA-fed shared-memory ring, double-buffered TMEM accumulators, persistent
// warp-specialised CTAs (warp 0 = TMA producer, warp 1 = MMA issuer, warps 2-5 = epilogue).
//
// Two tile engines, selected per call:
//   CG = 1: one CTA per 128x256 tile (UMMA 128x256x16, cta_group::1), 4 x 48 KB stages.
//   CG = 2: an SM pair (thread-block cluster of 2) per 256x256 tile (UMMA 256x256x16,
//           cta_group::2): each CTA stages its 128 rows of A and HALF of B, so the shared-
//           memory operand traffic per SM drops from 48 KB to 32 KB per k-block; the leader
//           CTA issues the MMAs and multicasts completion to both CTAs; 6 x 32 KB stages.
//
// Oracle it replaces: the per-expert numpy GEMMs of expert_activation / expert_forward
// (reference pkg/src/moelab/routing.py:59-68) and the GEMMs implied by the backward of
// combine_standard / combine_mem_efficient (routing.py:189-223).
//
// Two grouping modes, both driven by DEVICE-resident group metadata (no host sync):
//   grouped-M (fwd, dgrad): C[rows, N] = A[rows, K] * B_e^T where the expert-major
//     permuted activations are padded per expert to 128-row (CG=1) or 256-row (CG=2)
//     blocks, so every M tile belongs to exactly one expert (block_expert[] says which).
//   grouped-K (wgrad): C_e[M, N] = sum_{r in rows(e)} A[r, :M]^T B[r, :N] with the
//     reduction over the expert's (zero-padded) token rows.
//
// Epilogues (fused): plain bf16 store, fp32 store, SwiGLU (silu(gate)*up, optional
// per-row routing-prob scale for the memory-efficient combine), dSwiGLU (recompute
// phi from the saved pre-activation, optional prob scale + per-row dprob partials).
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace moe {
namespace gg {

constexpr int BM = 128;  // rows per CTA
constexpr int BN = 256;  // output columns per tile
constexpr int BK = 64;   // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int UMMA_K = 16;
constexpr int TMEM_COLS = 512;  // 2 accumulator stages x 256 fp32 columns
// Epilogue warps: 4 (one per TMEM lane quarter) or 8 (two per quarter, each owning half the
// tile's columns). Measured on B200: 8 warps did not speed up the dSwiGLU epilogue and cost
// ~13% on fc1+SwiGLU (the extra warps share the MMA issuer's SMSP), so 4 it is.
constexpr int EPI_WARPS = 4;
enum Epi : int { EPI_BF16 = 0, EPI_SWIGLU = 1, EPI_DSWIGLU = 2, EPI_F32 = 3 };
// The dSwiGLU epilogue (fc2 dgrad) reads the saved pre-activation and writes d_preact, 4
// bytes in and out per accumulator element plus the SwiGLU-backward math. In round 1 it
// kept the MMA issuer waiting on the accumulator release (ncu: 4.7M tempty spins per launch,
// tensor pipe 73%, 42 warp-instructions per element from the IEEE division;
// profiles/r02_ncu_gemm_mixtral_before.txt). With the fast-math sigmoid (dswiglu8) 4 warps
// (one per TMEM lane quarter) measured faster than 8 on B200: Mixtral fc2 dgrad 3.07 ms
// (1252 TFLOP/s) vs 3.61 ms, Qwen3 2.95 vs 3.20 ms. -DMOE_DSWIGLU_WARPS=8 rebuilds the other.
#ifndef MOE_DSWIGLU_WARPS
#define MOE_DSWIGLU_WARPS 4
#endif
constexpr int DSW_HALVES = MOE_DSWIGLU_WARPS / 4;  // dprob partials per (row, n-tile)
// dSwiGLU operands through shared memory: per epilogue warp and 32-column chunk, the gate /
// up pre-activation (32 rows x 32 columns each) arrive by TMA into a SWIZZLE_64B box one chunk
// ahead, d_gate / d_up overwrite them in place and leave by TMA tensor store (coalesced
// 64-byte row segments both ways instead of 16-byte per-thread accesses across 32 rows).
#ifndef MOE_DSWIGLU_TMA
#define MOE_DSWIGLU_TMA 1
#endif
constexpr int DSW_BOX = 32 * 32 * 2;                          // 32 rows x 32 bf16 columns
constexpr int DSW_STAGING = MOE_DSWIGLU_WARPS * 2 * 2 * DSW_BOX;  // warps x 2 bufs x (g, u)
// SwiGLU forward epilogue (fc1): gate / up pre-activation and act leave by TMA tensor stores
// of SWIZZLE_64B boxes (one (g, u, act) box set per epilogue warp) instead of 16-byte
// per-thread stores spread over 32 rows.
#ifndef MOE_SWIGLU_TMA
#define MOE_SWIGLU_TMA 1
#endif
// epilogue TMA traffic (preact / act / d_preact / dW boxes: streamed once) with an L2
// evict-first policy
#ifndef MOE_EPI_EVICT_FIRST
#define MOE_EPI_EVICT_FIRST 1
#endif
constexpr int SWG_STAGING = EPI_WARPS * 4 * DSW_BOX;  // per-warp stride of the dSwiGLU boxes
// Weight-gradient (grouped-K) kernels use 8 epilogue warps: with few token rows per expert
// (DeepSeek-shape EP=1: 128) each output tile has almost no MMA work and the kernel is a
// TMEM -> HBM drain, which 4 warps cannot keep busy.
template <bool GROUPED_K, int EPI>
constexpr int epi_warps() {
  return GROUPED_K ? 8 : (EPI == EPI_DSWIGLU ? MOE_DSWIGLU_WARPS : EPI_WARPS);
}
constexpr int BAND_M = 16;  // raster: 16 M units share each swept n-block (L2 reuse)

// SK: the small-K weight-gradient variant (few token rows per expert, e.g. DeepSeek-shape
// EP=1 with ~128): tiles are output-bound, so it trades operand stages for a 64 KB output
// staging area (two 4 KB TMA-store boxes per epilogue warp).
template <int CG, bool SK = false>
struct Cfg {
  static constexpr int A_STAGE = BM * BK * 2;           // this CTA's 128 rows of A
  static constexpr int B_ROWS = BN / CG;                // rows of the B tile this CTA stages
  static constexpr int B_STAGE = B_ROWS * BK * 2;
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int STAGES = SK ? (CG == 1 ? 3 : 4) : (CG == 1 ? 4 : 6);
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};
constexpr int SK_BOX_BYTES = 32 * 64 * 2;              // 32 rows x 64 bf16 columns
constexpr int SK_STAGING = 8 * 2 * SK_BOX_BYTES;       // 8 warps x double buffer
// Row-scatter epilogue (EPI_BF16, grouped-M, row_dst set): each epilogue warp stages its 32
// rows x 128 columns (half a tile row) in shared memory and writes every row with one
// 256-byte TMA bulk store to its destination (often a peer GPU over NVLink) instead of 16-B
// per-thread stores, which NVLink serves poorly.
// The weight-gradient kernels (8 epilogue warps) can use the same staged bulk stores for
// their local output rows (bulk_out; 64-column pieces, 128-byte rows).
constexpr int SCATTER_BYTES = 32 * 1024;  // staging for all epilogue warps
template <bool GROUPED_K>
constexpr int scatter_cols() { return GROUPED_K ? 64 : 128; }
template <int EPI, bool GROUPED_K, int CG, bool SK>
constexpr int smem_bytes() {
  // SK / dSwiGLU staging starts 1024-aligned after the barrier block (swizzled TMA boxes)
  return Cfg<CG, SK>::SMEM +
         (EPI == 0 ? (SK ? 768 + SK_STAGING : SCATTER_BYTES)
          : EPI == 2 ? (MOE_DSWIGLU_TMA ? 768 + DSW_STAGING : 0)
          : EPI == 1 ? (MOE_SWIGLU_TMA ? 768 + SWG_STAGING : 0)
                     : 0);
}


struct Params {
  // grouped-M
  const int* num_m_blocks;  // device scalar: active 128-row blocks
  const int* block_expert;  // [max_m_blocks]
  int max_m_blocks;
  // grouped-K
  const int* expert_offsets;  // [E+1], multiples of 64
  int num_experts;
  int M;  // grouped-K: output rows per expert
  int N;  // output columns (per expert), multiple of 256
  int K;  // grouped-M: reduction length, multiple of 64
  // epilogue operands
  void* out;
  long long ldo;
  long long out_expert_stride;
  void* out2;
  long long ldo2;
  const __nv_bfloat16* aux;
  long long ld_aux;
  const float* row_scale;
  float* row_partial;
  int ld_partial;
  // EPI_BF16 grouped-M scatter: absolute destination address of each output row (0 = drop
  // the row). Rows may live in peer GPUs' memory (NVLink): the EP combine / dX exchange is
  // fused into the producing GEMM's epilogue.
  const unsigned long long* row_dst;
  // EP dispatch overlap (grouped-M): source rank s's rows of the A operand are pushed over
  // NVLink while this GEMM runs; s then stores `epoch` into src_flag[s]. A tile's A rows are
  // loaded only once every source in block_need[128-row block] has signalled; units run in
  // unit_order (rows of early-arriving sources first). A 2 s timeout records wait_status
  // and traps (wait_sources).
  const uint32_t* src_flag;
  const uint32_t* epoch;  // device scalar (bumped in stream order before the dispatch)
  const uint32_t* block_need;
  const int* unit_order;
  int* wait_status;
  // epilogue outputs stored with the streaming (evict-first) cache hint, so the output
  // stream does not evict the operand tiles other CTAs still reuse from L2
  int stream_stores;
  int band_m;  // raster band: M units that sweep each n-block together (L2 reuse)
  int bulk_out;  // grouped-K EPI_BF16: the SK variant (TMA tensor stores of staged boxes)
  int debug_skip;  // SK diagnostics (MOE_B200_DEBUG_SKIP): 1 no epilogue work, 2 no output
                   // stores, 4 no MMAs (commits only); results are wrong when set
  int gk_mu_fast;  // grouped-K raster: M units fastest (when M < N), else n-blocks fastest
  // wave sync of the TMA producers (common.cuh wave_sync): off when sync_on == 0; sync points
  // at every tile start and, grouped-M only, every sync_kb k-blocks inside a tile (0 = none)
  int sync_on;
  int sync_slot;
  int sync_kb;
  int sync_lag;  // a producer at sync point g waits for every CTA to reach g - sync_lag
  // split units (grouped-M, kFlagSplit): unit u starts at 128-row block unit_block[u] and
  // *num_m_blocks counts UNITS (pairs for CG = 2, single blocks for CG = 1)
  const int* unit_block;
};

// per-(device, stream) wave-sync counters (common.cuh wave_sync_slot)
__device__ uint32_t g_wave_sync[kWaveSyncSlots * 32];

__device__ __forceinline__ void st_out(int4* p, int4 v, int cs) {
  if (cs)
    __stcs(p, v);
  else
    *p = v;
}

// Spin (bounded) until every source rank in `need` has published this epoch's rows. On a
// timeout (2 s) the kernel records [1, block, missing sources, epoch, flags[0..3]] in
// wait_status[0..7], makes it visible system-wide and traps: the launch fails with a CUDA
// error instead of multiplying rows that never arrived (check_ep_status() decodes the record).
__device__ __forceinline__ void wait_sources(const Params& p, uint32_t need, int blk,
                                             uint32_t epoch) {
  if (!need) return;
  const uint64_t t0 = globaltimer_ns();
  while (need) {
    const int s = __ffs(need) - 1;
    if (static_cast<int>(ld_acquire_sys_u32(p.src_flag + s) - epoch) >= 0) {
      need &= need - 1;
      continue;
    }
    if (globaltimer_ns() - t0 > 2000000000ull) {
      if (p.wait_status && atomicCAS(p.wait_status, 0, 1) == 0) {
        p.wait_status[1] = blk;
        p.wait_status[2] = static_cast<int>(need);
        p.wait_status[3] = static_cast<int>(epoch);
        for (int i = 0; i < 4; ++i)
          p.wait_status[4 + i] = static_cast<int>(ld_acquire_sys_u32(p.src_flag + i));
      }
      __threadfence_system();
      __trap();
    }
    __nanosleep(128);
  }
  fence_proxy_async_global();
}

struct Tile {
  int expert, m0, n0, k_begin, num_kb;
};

// Tile t of the cluster-level schedule; m0 is THIS CTA's first row (rank selects the half).
template <bool GROUPED_K, int CG>
__device__ __forceinline__ void decode_tile(const Params& p, int t, int num_units, int rank,
                                            Tile& tl) {
  const int nb_count = p.N / BN;
  if constexpr (!GROUPED_K) {
    // band_m <= 0: one expert's M units per band (clamped to [4, 16]); measured on B200
    // (profiles/r02_band_ab.txt): Qwen3 (8 units per expert) band 8 beats 16 by 3.7% over
    // the four grouped-M kinds, Mixtral (16 units per expert) band 16 beats 8
    int bm = p.band_m;
    if (bm <= 0) {
      bm = num_units / (p.num_experts > 0 ? p.num_experts : 1);
      bm = bm < 4 ? 4 : (bm > BAND_M ? BAND_M : bm);
    }
    const int band = t / (bm * nb_count);
    const int rem = t - band * bm * nb_count;
    const int u0 = band * bm;
    const int rows = min(bm, num_units - u0);
    const int nb = rem / rows;
    int u = u0 + (rem - nb * rows);
    if (p.unit_order) u = __ldg(p.unit_order + u);
    if (p.unit_block) {
      const int blk = __ldg(p.unit_block + u);
      tl.expert = __ldg(p.block_expert + blk);
      tl.m0 = blk * BM + rank * BM;
    } else {
      tl.expert = __ldg(p.block_expert + u * CG);
      tl.m0 = u * (BM * CG) + rank * BM;
    }
    tl.n0 = nb * BN;
    tl.k_begin = 0;
    tl.num_kb = p.K / BK;
  } else {
    const int mu_count = p.M / (BM * CG);
    const int per_e = mu_count * nb_count;
    const int e = t / per_e;
    const int rem = t - e * per_e;
    // raster within an expert: the fast index sweeps the operand whose per-expert slice is
    // the smaller one (it stays L2-resident while the other operand streams once)
    int mu, nb;
    if (p.gk_mu_fast) {
      nb = rem / mu_count;
      mu = rem - nb * mu_count;
    } else {
      mu = rem / nb_count;
      nb = rem - mu * nb_count;
    }
    tl.expert = e;
    tl.m0 = mu * (BM * CG) + rank * BM;
    tl.n0 = nb * BN;
    const int r0 = __ldg(p.expert_offsets + e);
    const int r1 = __ldg(p.expert_offsets + e + 1);
    tl.k_begin = r0;
    tl.num_kb = (r1 - r0) / BK;
  }
}

// Fast-math SwiGLU pieces for the epilogues: MUFU ex2 + MUFU rcp (rcp.approx.ftz, <= 1 ulp)
// instead of the IEEE division, whose refinement and slow-path checks made the dSwiGLU
// epilogue ~3x longer than the math needs. Saturates correctly: g -> -inf gives
// exp -> inf, rcp -> 0; g -> +inf gives exp -> 0, rcp -> 1. The outputs are bf16.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sigmoid_f(float g) { return rcp_approx(1.0f + __expf(-g)); }
__device__ __forceinline__ float silu_f(float g) { return g * sigmoid_f(g); }

// dSwiGLU of 8 accumulator columns: a = dL/d(act) (fp32), g / u = the saved gate / up
// pre-activations (bf16 x8 each). Writes d_gate = a*scale*u*s*(1 + g*(1-s)) and
// d_up = a*scale*silu(g) (bf16 x8 each); DP: also accumulates <a, silu(g)*u> (the dprob
// partial of the memory-efficient combine).
template <bool DP>
__device__ __forceinline__ void dswiglu8(const uint32_t* a, int4 gv, int4 uv, float scale,
                                         int4& dg_out, int4& du_out, float& dp) {
  const uint32_t* sg = reinterpret_cast<const uint32_t*>(&gv);
  const uint32_t* su = reinterpret_cast<const uint32_t*>(&uv);
  uint32_t* pg = reinterpret_cast<uint32_t*>(&dg_out);
  uint32_t* pu = reinterpret_cast<uint32_t*>(&du_out);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 gg = unpack_bf16x2(sg[j]);
    const float2 uu = unpack_bf16x2(su[j]);
    const float a0 = __uint_as_float(a[2 * j]), a1 = __uint_as_float(a[2 * j + 1]);
    const float s0 = sigmoid_f(gg.x), s1 = sigmoid_f(gg.y);
    const float si0 = gg.x * s0, si1 = gg.y * s1;
    if constexpr (DP) dp = fmaf(a0 * si0, uu.x, fmaf(a1 * si1, uu.y, dp));
    const float da0 = a0 * scale, da1 = a1 * scale;
    const float t0 = fmaf(gg.x, 1.0f - s0, 1.0f), t1 = fmaf(gg.y, 1.0f - s1, 1.0f);
    pg[j] = pack_bf16x2((da0 * uu.x) * (s0 * t0), (da1 * uu.y) * (s1 * t1));
    pu[j] = pack_bf16x2(da0 * si0, da1 * si1);
  }
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
// TMA load whose completion bytes land on the LEADER CTA's mbarrier (pair mode).
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const void* tmap,
                                                 uint64_t* bar, int x, int y) {
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;  // peer bit cleared -> CTA 0
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_leader), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Commit to the same-offset mbarrier in both CTAs of the pair.
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// Arrive on the leader CTA's copy of an mbarrier.
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

template <bool A_MN, bool B_MN, bool GROUPED_K, int EPI, int CG, bool SK>
__global__ void __launch_bounds__(64 + 32 * epi_warps<GROUPED_K, EPI>(), 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_b,
                        const __grid_constant__ CUtensorMap tmap_c,
                        const __grid_constant__ CUtensorMap tmap_d, const Params p) {
  using C = Cfg<CG, SK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::STAGES * C::A_STAGE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  // dSwiGLU operand boxes: 2 mbarriers per epilogue warp at +192 of the barrier block
  uint64_t* dsw_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE + 192);
  constexpr bool DSW_TMA = EPI == EPI_DSWIGLU && MOE_DSWIGLU_TMA;
  constexpr bool SWG_TMA = EPI == EPI_SWIGLU && MOE_SWIGLU_TMA;

  const int warp = warp_id();
  const int lane = lane_id();
  const int rank = CG == 2 ? static_cast<int>(cluster_rank()) : 0;
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], epi_warps<GROUPED_K, EPI>() * CG);
    }
    if constexpr (DSW_TMA || SWG_TMA) {
      tma_prefetch_desc(&tmap_c);
      tma_prefetch_desc(&tmap_d);
    }
    if constexpr (DSW_TMA) {
      for (int i = 0; i < 2 * epi_warps<GROUPED_K, EPI>(); ++i) mbar_init(&dsw_bar[i], 1);
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

  int num_tiles;
  int num_units = 0;
  if constexpr (!GROUPED_K) {
    num_units = p.unit_block ? *p.num_m_blocks : *p.num_m_blocks / CG;
    num_tiles = num_units * (p.N / BN);
  } else {
    num_tiles = p.num_experts * (p.M / (BM * CG)) * (p.N / BN);
  }
  // Allow a programmatic-dependent launch queued behind this grid (the split-unit tail
  // launch, which touches disjoint rows) to take SMs as soon as this grid's CTAs retire.
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int first = blockIdx.x / CG;
  const int stride = gridDim.x / CG;

  if (warp == 0) {
    // ===================== TMA producer (each CTA stages its own halves) ===============
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t epoch = p.src_flag ? *reinterpret_cast<const volatile uint32_t*>(p.epoch) : 0u;
      // wave sync: sync point (it, q) = phase q of this CTA's it-th tile, linear index
      // g = it * Q + q. Every CTA with a tile at iteration it arrives Q times there, so the
      // arrivals through g are CG * (it * S * Q + (q + 1) * P_it), P_it = CTA slots busy at
      // iteration it. A producer at g waits for the arrivals through g - lag (lag 0: a full
      // barrier; lag 1: nobody runs more than one phase ahead of the slowest CTA).
      uint32_t* wctr = p.sync_on ? g_wave_sync + p.sync_slot * 32 : nullptr;
      const int skb = GROUPED_K ? 0 : p.sync_kb;
      int it = 0;
      auto wsync = [&](int q, int num_kb) {
        const int nq = skb > 0 ? (num_kb + skb - 1) / skb : 1;
        const int g = it * nq + q - p.sync_lag;
        uint32_t target = 0;
        if (g >= 0) {
          const int it2 = g / nq, q2 = g - (g / nq) * nq;
          const int busy = min(stride, num_tiles - it2 * stride);
          target = static_cast<uint32_t>(CG * (it2 * stride * nq + (q2 + 1) * busy));
        }
        wave_sync(wctr, target, 100000ull);
      };
      for (int t = first; t < num_tiles; t += stride, ++it) {
        Tile tl;
        decode_tile<GROUPED_K, CG>(p, t, num_units, rank, tl);
        if (wctr) wsync(0, tl.num_kb);
        if constexpr (!GROUPED_K) {
          if (p.src_flag) wait_sources(p, __ldg(p.block_need + tl.m0 / BM), tl.m0 / BM, epoch);
        }
        for (int kb = 0; kb < tl.num_kb; ++kb) {
          if constexpr (!GROUPED_K) {
            if (wctr && skb > 0 && kb > 0 && kb % skb == 0) wsync(kb / skb, tl.num_kb);
          }
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full_bar[s], C::STAGE * CG);
          uint8_t* sa = smem_a + s * C::A_STAGE;
          uint8_t* sb = smem_b + s * C::B_STAGE;
          const int k = tl.k_begin + kb * BK;
          auto load = [&](void* dst, const CUtensorMap* tm, int x, int y) {
            if constexpr (CG == 1)
              tma_load_2d(dst, tm, &full_bar[s], x, y);
            else
              tma_load_2d_pair(dst, tm, &full_bar[s], x, y);
          };
          if constexpr (!A_MN) {
            load(sa, &tmap_a, k, tl.m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) load(sa + j * (64 * BK * 2), &tmap_a, tl.m0 + 64 * j, k);
          }
          const int nb0 = tl.n0 + rank * C::B_ROWS;
          if constexpr (!B_MN) {
            load(sb, &tmap_b, k, tl.expert * p.N + nb0);
          } else {
            const int krow = GROUPED_K ? k : tl.expert * p.K + k;
#pragma unroll
            for (int j = 0; j < C::B_ROWS / 64; ++j)
              load(sb + j * (64 * BK * 2), &tmap_b, nb0 + 64 * j, krow);
          }
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      if (wctr) wave_sync_exit(wctr);
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (single thread of the leader CTA) =================
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = make_idesc_bf16(BM * CG, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int t = first; t < num_tiles; t += stride) {
        Tile tl;
        decode_tile<GROUPED_K, CG>(p, t, num_units, rank, tl);
        if (tl.num_kb == 0) continue;
        mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < tl.num_kb; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem_a + s * C::A_STAGE);
          const uint32_t b_base = smem_u32(smem_b + s * C::B_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            const uint64_t adesc =
                A_MN ? make_sdesc_sw128(a_base + kk * (UMMA_K * 128), 64 * BK * 2, 1024)
                     : make_sdesc_sw128(a_base + kk * (UMMA_K * 2), 16, 1024);
            const uint64_t bdesc =
                B_MN ? make_sdesc_sw128(b_base + kk * (UMMA_K * 128), 64 * BK * 2, 1024)
                     : make_sdesc_sw128(b_base + kk * (UMMA_K * 2), 16, 1024);
            if (SK && (p.debug_skip & 4)) continue;
            if constexpr (CG == 1)
              umma_bf16(d_tmem, adesc, bdesc, idesc, (kb | kk) != 0 ? 1u : 0u);
            else
              umma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kb | kk) != 0 ? 1u : 0u);
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
        if (++acc == 2) {
          acc = 0;
          acc_ph ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue (warps 2..9: lane quarter x column half) ===========
    const int q = warp & 3;
    const int half = (warp - 2) / 4;
    constexpr int SC = scatter_cols<GROUPED_K>();
    uint8_t* stage = smem + C::STAGES * C::STAGE + 256 + (warp - 2) * (32 * SC * 2);
    // SK: two 4 KB boxes per warp, 1024-aligned; boxes alternate across the warp's pieces
    uint8_t* sk_box = smem + C::STAGES * C::STAGE + 1024 + (warp - 2) * (2 * SK_BOX_BYTES);
    int sk_piece = 0;
    constexpr int EC = BN / (epi_warps<GROUPED_K, EPI>() / 4);  // tile columns per epilogue warp
    const int cb = half * EC;  // this warp's first tile column
    const int row_local = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    int acc = 0;
    uint32_t acc_ph = 0;
    // dSwiGLU boxes of this warp: buffer b holds gate at +0 and up at +DSW_BOX
    uint8_t* dsw_buf = smem + C::STAGES * C::STAGE + 1024 + (warp - 2) * (4 * DSW_BOX);
    uint64_t* dbar = dsw_bar + (warp - 2) * 2;
    const uint64_t epi_pol = l2_evict_first_policy();
    uint32_t dsw_ph = 0;  // bit b: parity of buffer b's next completion
    int dsw_seq = 0;      // chunks consumed by this warp (buffer = dsw_seq & 1)
    auto dsw_load = [&](const Tile& tn, int c, int b) {
      const int j0 = tn.n0 + cb + c * 32;
      const int gpos = (j0 >> 7) * 256 + (j0 & 127);
      const int y = tn.m0 + q * 32;
      uint8_t* dst = dsw_buf + b * (2 * DSW_BOX);
      mbar_arrive_expect_tx(&dbar[b], 2 * DSW_BOX);
      if (MOE_EPI_EVICT_FIRST) {
        tma_load_2d_hint(dst, &tmap_d, &dbar[b], gpos, y, epi_pol);
        tma_load_2d_hint(dst + DSW_BOX, &tmap_d, &dbar[b], gpos + 128, y, epi_pol);
      } else {
        tma_load_2d(dst, &tmap_d, &dbar[b], gpos, y);
        tma_load_2d(dst + DSW_BOX, &tmap_d, &dbar[b], gpos + 128, y);
      }
    };
    if constexpr (DSW_TMA) {
      if (first < num_tiles && lane == 0) {
        Tile t0;
        decode_tile<GROUPED_K, CG>(p, first, num_units, rank, t0);
        dsw_load(t0, 0, 0);
      }
    }
    for (int t = first; t < num_tiles; t += stride) {
      Tile tl;
      decode_tile<GROUPED_K, CG>(p, t, num_units, rank, tl);
      const long long row = tl.m0 + row_local;
      if (tl.num_kb == 0) {
        // Expert with no rows: its weight gradient is exactly zero.
        if constexpr (EPI == EPI_BF16) {
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) +
                             tl.expert * p.out_expert_stride + row * p.ldo + tl.n0 + cb;
          const int4 z = make_int4(0, 0, 0, 0);
#pragma unroll 4
          for (int c = 0; c < EC / 8; ++c) reinterpret_cast<int4*>(o)[c] = z;
        } else if constexpr (EPI == EPI_F32) {
          float* o = reinterpret_cast<float*>(p.out) + tl.expert * p.out_expert_stride +
                     row * p.ldo + tl.n0 + cb;
          const int4 z = make_int4(0, 0, 0, 0);
#pragma unroll 4
          for (int c = 0; c < EC / 4; ++c) reinterpret_cast<int4*>(o)[c] = z;
        }
        continue;
      }
      // dSwiGLU: the first chunk's pre-activation (DRAM/L2 latency) is fetched while the
      // tile's MMAs are still running; later chunks are prefetched one chunk ahead.
      int4 pre_g[4], pre_u[4];
      if constexpr (EPI == EPI_DSWIGLU && !DSW_TMA) {
        const __nv_bfloat16* pr = p.aux + row * p.ld_aux;
        const int jc = tl.n0 + cb;
        const long long pos0 = (long long)(jc >> 7) * 256 + (jc & 127);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          pre_g[v] = reinterpret_cast<const int4*>(pr + pos0)[v];
          pre_u[v] = reinterpret_cast<const int4*>(pr + pos0 + 128)[v];
        }
      }
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
      const uint32_t t_base = tmem_base + lane_off + acc * BN;

      if constexpr (EPI == EPI_BF16 && GROUPED_K && SK) {
        // 64-column pieces: this warp's 32 rows x 64 columns go to a SWIZZLE_128B box in
        // shared memory (lane = row; 16-byte chunk j stored at j ^ (row & 7): the 16-byte
        // stores of a warp hit distinct bank groups) and leave with one TMA tensor store; two
        // boxes alternate so a store drains while the next piece is staged. Both 32-column
        // TMEM loads of a piece are in flight before the single wait.
#pragma unroll 1
        for (int pc = 0; pc < (p.debug_skip & 1 ? 0 : EC / 64); ++pc) {
          const int col = cb + pc * 64;
          uint32_t r[2][32];
          tmem_ld_32x32b_x32(t_base + col, r[0]);
          tmem_ld_32x32b_x32(t_base + col + 32, r[1]);
          uint8_t* box = sk_box + (sk_piece & 1) * SK_BOX_BYTES;
          if (lane == 0) bulk_wait_read_1();  // the store that last used this box has read it
          __syncwarp();
          tmem_ld_wait();
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const uint32_t* rv = r[v >> 2] + 8 * (v & 3);
            int4 w;
            w.x = pack_bf16x2(__uint_as_float(rv[0]), __uint_as_float(rv[1]));
            w.y = pack_bf16x2(__uint_as_float(rv[2]), __uint_as_float(rv[3]));
            w.z = pack_bf16x2(__uint_as_float(rv[4]), __uint_as_float(rv[5]));
            w.w = pack_bf16x2(__uint_as_float(rv[6]), __uint_as_float(rv[7]));
            *reinterpret_cast<int4*>(box + lane * 128 + ((v ^ (lane & 7)) * 16)) = w;
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0 && !(p.debug_skip & 2)) {
            if (MOE_EPI_EVICT_FIRST)
              tma_store_2d_hint(&tmap_c, box, tl.n0 + col, tl.expert * p.M + tl.m0 + q * 32,
                                epi_pol);
            else
              tma_store_2d(&tmap_c, box, tl.n0 + col, tl.expert * p.M + tl.m0 + q * 32);
            bulk_commit();
          }
          ++sk_piece;
        }
      } else if constexpr (EPI == EPI_BF16 || EPI == EPI_F32) {
        const long long ebase = GROUPED_K ? tl.expert * p.out_expert_stride : 0;
#pragma unroll 1
        for (int c = 0; c < EC / 32; ++c) {
          const int col = cb + c * 32;
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_base + col, r);
          tmem_ld_wait();
          if constexpr (EPI == EPI_BF16) {
            if (!GROUPED_K && p.row_dst) {
              // stage this lane's row chunk; one bulk store per (row, SC columns)
              const int hc = col % SC;
              uint8_t* srow = stage + lane * (SC * 2);
              if (hc == 0) bulk_wait_read_all();  // slot free again (previous half read)
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                int4 w;
                w.x = pack_bf16x2(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1]));
                w.y = pack_bf16x2(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3]));
                w.z = pack_bf16x2(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5]));
                w.w = pack_bf16x2(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7]));
                reinterpret_cast<int4*>(srow + hc * 2)[v] = w;
              }
              if (hc + 32 == SC) {
                const unsigned long long dst = __ldg(p.row_dst + row);
                fence_async_shared();
                if (dst) {
                  bulk_store_s2g(reinterpret_cast<__nv_bfloat16*>(dst) + tl.n0 + col + 32 - SC,
                                 srow, SC * 2);
                  bulk_commit();
                }
              }
              continue;
            }
            __nv_bfloat16* o =
                reinterpret_cast<__nv_bfloat16*>(p.out) + ebase + row * p.ldo + tl.n0 + col;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              int4 w;
              w.x = pack_bf16x2(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1]));
              w.y = pack_bf16x2(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3]));
              w.z = pack_bf16x2(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5]));
              w.w = pack_bf16x2(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7]));
              st_out(reinterpret_cast<int4*>(o) + v, w, p.stream_stores);
            }
          } else {
            float* o = reinterpret_cast<float*>(p.out) + ebase + row * p.ldo + tl.n0 + col;
#pragma unroll
            for (int v = 0; v < 8; ++v)
              st_out(reinterpret_cast<int4*>(o) + v,
                     make_int4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]),
                     p.stream_stores);
          }
        }
      } else if constexpr (SWG_TMA) {
        // Tile columns [0,128) = gate rows, [128,256) = up rows of the interleaved W1; 32
        // gate columns and the matching up columns per chunk -> (g, u, act) boxes.
        const float scale = p.row_scale ? __ldg(p.row_scale + row) : 1.0f;
        const int sw = (lane >> 1) & 3;  // SWIZZLE_64B
        uint8_t* box = dsw_buf;          // this warp's 3 boxes: g, u, act
        uint8_t* grow = box + lane * 64;
#pragma unroll 1
        for (int c = 0; c < EC / 64; ++c) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(t_base + (cb >> 1) + c * 32, g);
          tmem_ld_32x32b_x32(t_base + 128 + (cb >> 1) + c * 32, u);
          if (lane == 0) bulk_wait_read_0();  // the previous chunk's stores have read the boxes
          __syncwarp();
          tmem_ld_wait();
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            int4 wg, wu, wa;
            uint32_t* pg = reinterpret_cast<uint32_t*>(&wg);
            uint32_t* pu = reinterpret_cast<uint32_t*>(&wu);
            uint32_t* pa = reinterpret_cast<uint32_t*>(&wa);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = 8 * v + 2 * j;
              const float g0 = __uint_as_float(g[i]), g1 = __uint_as_float(g[i + 1]);
              const float u0 = __uint_as_float(u[i]), u1 = __uint_as_float(u[i + 1]);
              pg[j] = pack_bf16x2(g0, g1);
              pu[j] = pack_bf16x2(u0, u1);
              pa[j] = pack_bf16x2(silu_f(g0) * u0 * scale, silu_f(g1) * u1 * scale);
            }
            const int off = (v ^ sw) << 4;
            *reinterpret_cast<int4*>(grow + off) = wg;
            *reinterpret_cast<int4*>(grow + DSW_BOX + off) = wu;
            *reinterpret_cast<int4*>(grow + 2 * DSW_BOX + off) = wa;
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            const int x = tl.n0 + (cb >> 1) + c * 32;
            const int y = tl.m0 + q * 32;
            if (MOE_EPI_EVICT_FIRST) {
              tma_store_2d_hint(&tmap_c, box, x, y, epi_pol);
              tma_store_2d_hint(&tmap_c, box + DSW_BOX, x + 128, y, epi_pol);
              tma_store_2d_hint(&tmap_d, box + 2 * DSW_BOX, (tl.n0 >> 1) + (cb >> 1) + c * 32, y,
                                epi_pol);
            } else {
              tma_store_2d(&tmap_c, box, x, y);
              tma_store_2d(&tmap_c, box + DSW_BOX, x + 128, y);
              tma_store_2d(&tmap_d, box + 2 * DSW_BOX, (tl.n0 >> 1) + (cb >> 1) + c * 32, y);
            }
            bulk_commit();
          }
        }
      } else if constexpr (EPI == EPI_SWIGLU) {
        // Tile columns [0,128) = gate rows, [128,256) = up rows of the interleaved W1; this
        // warp takes gate columns [half*64, +64) and the matching up columns.
        const float scale = p.row_scale ? __ldg(p.row_scale + row) : 1.0f;
        __nv_bfloat16* pre =
            reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.ldo + tl.n0 + (cb >> 1);
        __nv_bfloat16* act =
            reinterpret_cast<__nv_bfloat16*>(p.out2) + row * p.ldo2 + (tl.n0 >> 1) + (cb >> 1);
#pragma unroll 1
        for (int c = 0; c < EC / 64; ++c) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(t_base + (cb >> 1) + c * 32, g);
          tmem_ld_32x32b_x32(t_base + 128 + (cb >> 1) + c * 32, u);
          tmem_ld_wait();
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            int4 wg, wu, wa;
            uint32_t* pg = reinterpret_cast<uint32_t*>(&wg);
            uint32_t* pu = reinterpret_cast<uint32_t*>(&wu);
            uint32_t* pa = reinterpret_cast<uint32_t*>(&wa);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = 8 * v + 2 * j;
              const float g0 = __uint_as_float(g[i]), g1 = __uint_as_float(g[i + 1]);
              const float u0 = __uint_as_float(u[i]), u1 = __uint_as_float(u[i + 1]);
              pg[j] = pack_bf16x2(g0, g1);
              pu[j] = pack_bf16x2(u0, u1);
              pa[j] = pack_bf16x2(silu_f(g0) * u0 * scale, silu_f(g1) * u1 * scale);
            }
            st_out(reinterpret_cast<int4*>(pre + c * 32) + v, wg, p.stream_stores);
            st_out(reinterpret_cast<int4*>(pre + 128 + c * 32) + v, wu, p.stream_stores);
            st_out(reinterpret_cast<int4*>(act + c * 32) + v, wa, p.stream_stores);
          }
        }
      } else if constexpr (DSW_TMA) {
        // Accumulator = dL/d(act) (or dL/d(p*act) for the mem-efficient combine) for this
        // warp's columns of the m-wide activation; phi is recomputed from the preact box.
        const float scale = p.row_scale ? __ldg(p.row_scale + row) : 1.0f;
        float dp_acc = 0.0f;
        const int sw = (lane >> 1) & 3;  // SWIZZLE_64B: 16-byte chunk j of row r at j ^ sw
#pragma unroll 1
        for (int c = 0; c < EC / 32; ++c) {
          const int b = dsw_seq & 1;
          if (lane == 0) {
            // next chunk (this tile, or chunk 0 of this warp's next tile) into the other box,
            // once the store that last read that box has drained
            bulk_wait_read_0();
            if (c + 1 < EC / 32) {
              dsw_load(tl, c + 1, b ^ 1);
            } else if (t + stride < num_tiles) {
              Tile tn;
              decode_tile<GROUPED_K, CG>(p, t + stride, num_units, rank, tn);
              dsw_load(tn, 0, b ^ 1);
            }
          }
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_base + cb + c * 32, r);
          mbar_wait(&dbar[b], (dsw_ph >> b) & 1);
          dsw_ph ^= 1u << b;
          tmem_ld_wait();
          uint8_t* gbox = dsw_buf + b * (2 * DSW_BOX) + lane * 64;
          uint8_t* ubox = gbox + DSW_BOX;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            int4* gp = reinterpret_cast<int4*>(gbox + ((v ^ sw) << 4));
            int4* up = reinterpret_cast<int4*>(ubox + ((v ^ sw) << 4));
            int4 wg, wu;
            if (p.row_partial)
              dswiglu8<true>(r + 8 * v, *gp, *up, scale, wg, wu, dp_acc);
            else
              dswiglu8<false>(r + 8 * v, *gp, *up, scale, wg, wu, dp_acc);
            *gp = wg;
            *up = wu;
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            const int j0 = tl.n0 + cb + c * 32;
            const int gpos = (j0 >> 7) * 256 + (j0 & 127);
            const int y = tl.m0 + q * 32;
            uint8_t* box = dsw_buf + b * (2 * DSW_BOX);
            if (MOE_EPI_EVICT_FIRST) {
              tma_store_2d_hint(&tmap_c, box, gpos, y, epi_pol);
              tma_store_2d_hint(&tmap_c, box + DSW_BOX, gpos + 128, y, epi_pol);
            } else {
              tma_store_2d(&tmap_c, box, gpos, y);
              tma_store_2d(&tmap_c, box + DSW_BOX, gpos + 128, y);
            }
            bulk_commit();
          }
          ++dsw_seq;
        }
        if (p.row_partial)
          p.row_partial[row * p.ld_partial + (tl.n0 / BN) * DSW_HALVES + half] = dp_acc;
      } else if constexpr (EPI == EPI_DSWIGLU) {
        // Accumulator = dL/d(act) (or dL/d(p*act) for the mem-efficient combine) for
        // columns [n0, n0+256) of the m-wide activation. Recompute phi from preact.
        const float scale = p.row_scale ? __ldg(p.row_scale + row) : 1.0f;
        float dp_acc = 0.0f;
        const __nv_bfloat16* pre_row = p.aux + row * p.ld_aux;
        __nv_bfloat16* dpre_row = reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.ldo;
#pragma unroll 1
        for (int c = 0; c < EC / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_base + cb + c * 32, r);
          const int j0 = tl.n0 + cb + c * 32;
          const long long pos = (long long)(j0 >> 7) * 256 + (j0 & 127);
          int4 gv[4], uv[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            gv[v] = pre_g[v];
            uv[v] = pre_u[v];
          }
          if (c + 1 < EC / 32) {  // prefetch the next chunk's pre-activation
            const int j1 = j0 + 32;
            const long long pos1 = (long long)(j1 >> 7) * 256 + (j1 & 127);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              pre_g[v] = reinterpret_cast<const int4*>(pre_row + pos1)[v];
              pre_u[v] = reinterpret_cast<const int4*>(pre_row + pos1 + 128)[v];
            }
          }
          tmem_ld_wait();
          if (p.row_partial) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              int4 wg, wu;
              dswiglu8<true>(r + 8 * v, gv[v], uv[v], scale, wg, wu, dp_acc);
              st_out(reinterpret_cast<int4*>(dpre_row + pos) + v, wg, p.stream_stores);
              st_out(reinterpret_cast<int4*>(dpre_row + pos + 128) + v, wu, p.stream_stores);
            }
          } else {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              int4 wg, wu;
              dswiglu8<false>(r + 8 * v, gv[v], uv[v], scale, wg, wu, dp_acc);
              st_out(reinterpret_cast<int4*>(dpre_row + pos) + v, wg, p.stream_stores);
              st_out(reinterpret_cast<int4*>(dpre_row + pos + 128) + v, wu, p.stream_stores);
            }
          }
        }
        if (p.row_partial)
          p.row_partial[row * p.ld_partial + (tl.n0 / BN) * DSW_HALVES + half] = dp_acc;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1)
          mbar_arrive(&tempty_bar[acc]);
        else
          mbar_arrive_leader(&tempty_bar[acc]);
      }
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
  }

  // scattered rows may be in peer memory: complete the bulk stores and make them visible
  // system-wide before the stream-ordered collective that publishes them
  if ((DSW_TMA || SWG_TMA ||
       (EPI == EPI_BF16 && ((!GROUPED_K && p.row_dst) || (GROUPED_K && SK)))) &&
      warp >= 2) {
    bulk_wait_all();
    __threadfence_system();
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
  // A programmatic-dependent grid (the split-unit tail) completes only after the grid it
  // overlapped, so work queued behind it sees both. No-op for a normal launch.
  if (threadIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ------------------------------------------------------------------ host side

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

// 2-D bf16 tensor [outer, inner] with row stride `ld` elements, 128B-swizzled boxes.
static int make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                     uint64_t ld, uint32_t box_inner, uint32_t box_outer,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return kErrCuda;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * 2) & 15)) return kErrInvalidArg;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? kOk : kErrCuda;
}

static int num_sms() { return device_sms(); }

template <bool A_MN, bool B_MN, bool GROUPED_K, int EPI, int CG, bool SK>
static int launch_cg(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                     const CUtensorMap& td, const Params& p, int max_tiles,
                     cudaStream_t stream, bool pdl = false) {
  auto kern = grouped_gemm_kernel<A_MN, B_MN, GROUPED_K, EPI, CG, SK>;
  MOE_CUDA_CHECK(ensure_dyn_smem(reinterpret_cast<const void*>(kern),
                                 smem_bytes<EPI, GROUPED_K, CG, SK>()));
  if (max_tiles <= 0) return kOk;
  int grid = max_tiles * CG < num_sms() ? max_tiles * CG : num_sms();
  grid -= grid % CG;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64 + 32 * epi_warps<GROUPED_K, EPI>());
  cfg.dynamicSmemBytes = smem_bytes<EPI, GROUPED_K, CG, SK>();
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  MOE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, td, p));
  return kOk;
}

// flags bit 0: CTA-pair engine (grouped-M: expert blocks 256-row aligned).
constexpr int kFlagPair = 1;
// flags bit 1: split units (with bit 0): num_m_blocks is the unit table of moe_split_units
// over a 128-row aligned plan; pairs run on the CTA-pair engine, single blocks on the 1-CTA
// engine (two launches). Not with the EP source waits.
constexpr int kFlagSplit = 2;

// Builds tensor maps for the chosen engine and launches. a_inner/a_outer/b_* describe the
// 2-D global views; a/b K-major (box {64, rows}) or MN-major (box {64, 64}).
static int stream_stores_default() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_B200_EPI_CS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}

template <bool A_MN, bool B_MN, bool GROUPED_K, int EPI>
static int run(const void* a, uint64_t a_inner, uint64_t a_outer, const void* b,
               uint64_t b_inner, uint64_t b_outer, Params p, int units_m, int pair,
               cudaStream_t stream, int split = 0, int pdl_launch = 0) {
  p.stream_stores = stream_stores_default();
  {
    static int bm = -1;  // MOE_B200_BAND forces a band; else auto (pair) / BAND_M (1-CTA)
    if (bm < 0) {
      const char* e = getenv("MOE_B200_BAND");
      bm = e ? atoi(e) : 0;
      if (bm < 0) bm = 0;
    }
    p.band_m = bm > 0 ? bm : (pair ? 0 : BAND_M);
  }
  {
    // grouped-K with few token rows per expert (avg <= 512: DeepSeek-shape EP=1 has 128) is
    // output-bound: the SK variant (staged boxes + TMA tensor stores). With long K the
    // per-thread stores of the 6-stage engine are as fast (Mixtral, Qwen3).
    static int bo = -2;
    if (bo == -2) {
      const char* e = getenv("MOE_B200_WGRAD_BULK");
      bo = e ? (e[0] == '1' ? 1 : 0) : -1;
    }
    const long long avg_k = p.num_experts > 0 ? (long long)a_outer / p.num_experts : 0;
    p.bulk_out = bo >= 0 ? bo : (GROUPED_K && avg_k > 0 && avg_k <= 512 ? 1 : 0);
    // Mixtral dW2 (M = h = 4096 < N = m = 14336): sweeping the 256-column n-blocks fastest
    // kept the whole per-expert act slice (117 MB) in flight and re-read it from DRAM for
    // every M unit (ncu: 11.4 GB for 2.1 GB algorithmic); M units fastest keeps the 34 MB
    // d_O slice resident instead. MOE_B200_GK_RASTER=mu|nb forces one order.
    static int gr = -2;
    if (gr == -2) {
      const char* e = getenv("MOE_B200_GK_RASTER");
      gr = e ? (e[0] == 'm' ? 1 : 0) : -1;
    }
    p.gk_mu_fast = GROUPED_K ? (gr >= 0 ? gr : (p.M < p.N ? 1 : 0)) : 0;
  }
  {
    // wave sync of the producers (common.cuh wave_sync). MOE_B200_WAVE_SYNC=0 turns it off;
    // MOE_B200_SYNC_KB sets the in-tile sync period (k-blocks, grouped-M; 0 = tile starts only)
    static int on = -1, kb = -1, lag = 0, min_kb = 0;
    if (on < 0) {
      const char* e = getenv("MOE_B200_WAVE_SYNC");
      on = (e && e[0] == '0') ? 0 : 1;
      const char* k = getenv("MOE_B200_SYNC_KB");
      kb = k ? atoi(k) : 32;
      if (kb < 0) kb = 0;
      const char* l = getenv("MOE_B200_SYNC_LAG");
      lag = l ? atoi(l) : 1;
      if (lag < 0) lag = 0;
      const char* m = getenv("MOE_B200_SYNC_MIN_KB");
      min_kb = m ? atoi(m) : 256;
    }
    // Measured on B200 (profiles/r02_wave_sync.txt): the sync cuts DRAM reads (Mixtral fc1
    // dgrad 15.5 -> 10.3 GB, dW1 5.0 -> 2.6 GB) and raises the power-capped clock, but its
    // waits cost more than that wins except on very long K (Mixtral fc1 dgrad, K = 28672:
    // 6.05 -> 5.88 ms with 32-k-block phases, lag 1). Default: grouped-M only, K >= 256
    // k-blocks. Grouped-K (weight gradients) measured slower with it at every setting.
    const bool want = on && !GROUPED_K && p.K / BK >= min_kb;
    p.sync_slot = want ? wave_sync_slot(stream) : -1;
    p.sync_on = p.sync_slot >= 0 ? 1 : 0;
    p.sync_kb = kb;
    p.sync_lag = lag;
  }
  CUtensorMap ta, tb, tc, td;
  int st;
  const int cg = pair ? 2 : 1;
  if ((st = make_tmap(&ta, a, a_inner, a_outer, a_inner, 64, A_MN ? BK : BM))) return st;
  if ((st = make_tmap(&tb, b, b_inner, b_outer, b_inner, 64, B_MN ? BK : BN / cg))) return st;
  const int nb = p.N / BN;
  if constexpr (GROUPED_K && EPI == EPI_BF16) {
    if (p.bulk_out) {
      // output dW [E*M rows, N] bf16, boxes of 32 rows x 64 columns, SWIZZLE_128B
      if ((st = make_tmap(&tc, p.out, p.N, (uint64_t)p.num_experts * p.M, p.ldo, 64, 32)))
        return st;
      if (pair)
        return launch_cg<A_MN, B_MN, true, EPI, 2, true>(ta, tb, tc, tc, p, (units_m / 2) * nb,
                                                         stream, pdl_launch != 0);
      return launch_cg<A_MN, B_MN, true, EPI, 1, true>(ta, tb, tc, tc, p, units_m * nb, stream,
                                                       pdl_launch != 0);
    }
  }
  tc = tb;  // unused by the other variants
  td = tb;
  if constexpr (EPI == EPI_SWIGLU && MOE_SWIGLU_TMA) {
    // preact [rows, 2m] and act [rows, m] bf16 (stores), 32 x 32 boxes, SWIZZLE_64B
    const uint64_t rows = (uint64_t)p.max_m_blocks * BM;
    if ((st = make_tmap(&tc, p.out, p.ldo, rows, p.ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)))
      return st;
    if ((st = make_tmap(&td, p.out2, p.ldo2, rows, p.ldo2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)))
      return st;
  }
  if constexpr (EPI == EPI_DSWIGLU && MOE_DSWIGLU_TMA) {
    // d_preact (store) and preact (load): [rows, 2m] bf16, 32 x 32 boxes, SWIZZLE_64B
    const uint64_t rows = (uint64_t)p.max_m_blocks * BM;
    if ((st = make_tmap(&tc, p.out, p.ldo, rows, p.ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)))
      return st;
    if ((st = make_tmap(&td, p.aux, p.ld_aux, rows, p.ld_aux, 32, 32,
                        CU_TENSOR_MAP_SWIZZLE_64B)))
      return st;
  }
  if constexpr (!GROUPED_K) {
    if (split) {
      // kFlagSplit: num_m_blocks points at the unit table U of moe_split_units (a 128-row
      // aligned plan): U[0] pairs, U[1] singles, U[2..2+cap) pair start blocks,
      // U[2+cap..2+2cap) single blocks. The 256-row pairs run on the CTA-pair engine, each
      // expert's odd last block on the 1-CTA engine (half the padding of a 256-row plan).
      const int* U = p.num_m_blocks;
      const int cap = p.max_m_blocks;
      Params pp = p;
      pp.unit_block = U + 2;
      pp.num_m_blocks = U;
      int st2 = launch_cg<A_MN, B_MN, GROUPED_K, EPI, 2, false>(ta, tb, tc, td, pp,
                                                                 (cap / 2) * nb, stream);
      if (st2) return st2;
      CUtensorMap tb1 = tb;  // the 1-CTA engine stages all 256 B rows
      if (!B_MN && (st2 = make_tmap(&tb1, b, b_inner, b_outer, b_inner, 64, BN))) return st2;
      Params ps = p;
      ps.unit_block = U + 2 + cap;
      ps.num_m_blocks = U + 1;
      const int singles = p.num_experts < cap ? p.num_experts : cap;
      // programmatic dependent launch: the tail tiles take the SMs the pair grid's last
      // wave leaves idle (disjoint rows, no data dependency; the next launch on the stream
      // still waits for both). Its own wave sync would share the stream's counter: off.
      static int pdl = -1;
      if (pdl < 0) {
        const char* e = getenv("MOE_B200_SPLIT_PDL");
        pdl = (e && e[0] == '0') ? 0 : 1;
      }
      if (pdl) {
        ps.sync_on = 0;
        ps.sync_slot = -1;
      }
      return launch_cg<A_MN, B_MN, GROUPED_K, EPI, 1, false>(ta, tb1, tc, td, ps, singles * nb,
                                                             stream, pdl != 0);
    }
  }
  if (pair)
    return launch_cg<A_MN, B_MN, GROUPED_K, EPI, 2, false>(ta, tb, tc, td, p,
                                                           (units_m / 2) * nb, stream,
                                                           pdl_launch != 0);
  return launch_cg<A_MN, B_MN, GROUPED_K, EPI, 1, false>(ta, tb, tc, td, p, units_m * nb,
                                                         stream, pdl_launch != 0);
}

}  // namespace gg
}  // namespace moe

using namespace moe;
using namespace moe::gg;

extern "C" {

// fc1 forward + SwiGLU.  xp[rows, h] (expert-major, padded plan), w1[E, 2m, h] with
// gate/up interleaved in 128-row blocks.  Writes preact[rows, 2m] (interleaved) and
// act[rows, m] = silu(gate) * up (* row_prob[row] when row_prob != NULL).
// a_rows: physical rows of xp (TMA bound; rows beyond read as zero), max_rows: rows of the
// output buffers (multiple of 128; of 256 with the pair flag).
struct SourceWait {
  const uint32_t* src_flag;
  const uint32_t* epoch;  // device scalar (bumped in stream order before the dispatch)
  const uint32_t* block_need;
  const int* unit_order;
  int* status;
};
static void set_wait(Params& p, const SourceWait* w) {
  if (!w) return;
  p.src_flag = w->src_flag;
  p.epoch = w->epoch;
  p.block_need = w->block_need;
  p.unit_order = w->unit_order;
  p.wait_status = w->status;
}

static int fc1_fwd_impl(const void* xp, const void* w1, int a_rows, int max_rows, int h, int m,
                        int num_experts, const int* block_expert, const int* num_m_blocks,
                        const float* row_prob, void* preact, void* act, int flags,
                        const SourceWait* w, void* stream) {
  const int pair = flags & kFlagPair;
  const int split = (flags & kFlagSplit) && pair;
  if (h % BK || (2 * m) % BN || max_rows % (BM * (pair && !split ? 2 : 1)) ||
      a_rows > max_rows || (split && w))
    return kErrInvalidArg;
  Params p{};
  set_wait(p, w);
  p.num_m_blocks = num_m_blocks;
  p.block_expert = block_expert;
  p.max_m_blocks = max_rows / BM;
  p.num_experts = num_experts;
  p.N = 2 * m;
  p.K = h;
  p.out = preact;
  p.ldo = 2 * m;
  p.out2 = act;
  p.ldo2 = m;
  p.row_scale = row_prob;
  return run<false, false, false, EPI_SWIGLU>(xp, h, a_rows, w1, h, (uint64_t)num_experts * 2 * m,
                                              p, p.max_m_blocks, pair,
                                              static_cast<cudaStream_t>(stream), split);
}

int moe_gg_fc1_fwd(const void* xp, const void* w1, int a_rows, int max_rows, int h, int m,
                   int num_experts, const int* block_expert, const int* num_m_blocks,
                   const float* row_prob, void* preact, void* act, int flags, void* stream) {
  return fc1_fwd_impl(xp, w1, a_rows, max_rows, h, m, num_experts, block_expert, num_m_blocks,
                      row_prob, preact, act, flags, nullptr, stream);
}

// fc1 forward overlapped with the EP dispatch: tiles wait for their rows' source ranks
// (src_flag[s] >= epoch, written by moe_ep_signal after each source's push) and run in
// unit_order. block_need[128-row block] = bitmask of source ranks.
int moe_gg_fc1_fwd_ep(const void* xp, const void* w1, int a_rows, int max_rows, int h, int m,
                      int num_experts, const int* block_expert, const int* num_m_blocks,
                      const float* row_prob, void* preact, void* act, int flags,
                      const unsigned int* src_flag, const unsigned int* epoch,
                      const unsigned int* block_need, const int* unit_order, int* status,
                      void* stream) {
  if (!src_flag || !epoch || !block_need) return kErrInvalidArg;
  const SourceWait w{src_flag, epoch, block_need, unit_order, status};
  return fc1_fwd_impl(xp, w1, a_rows, max_rows, h, m, num_experts, block_expert, num_m_blocks,
                      row_prob, preact, act, flags, &w, stream);
}

static int fc2_fwd_impl(const void* act, const void* w2, int a_rows, int max_rows, int m,
                        int h, int num_experts, const int* block_expert,
                        const int* num_m_blocks, void* out, const unsigned long long* row_dst,
                        int flags, void* stream) {
  const int pair = flags & kFlagPair;
  const int split = (flags & kFlagSplit) && pair;
  if (m % BK || h % BN || max_rows % (BM * (pair && !split ? 2 : 1)) || a_rows > max_rows)
    return kErrInvalidArg;
  Params p{};
  p.row_dst = row_dst;
  p.num_m_blocks = num_m_blocks;
  p.block_expert = block_expert;
  p.max_m_blocks = max_rows / BM;
  p.num_experts = num_experts;
  p.N = h;
  p.K = m;
  p.out = out;
  p.ldo = h;
  return run<false, false, false, EPI_BF16>(act, m, a_rows, w2, m, (uint64_t)num_experts * h, p,
                                            p.max_m_blocks, pair,
                                            static_cast<cudaStream_t>(stream), split);
}

// fc2 forward: out[rows, h] = act[rows, m] * w2_e^T, w2[E, h, m].
int moe_gg_fc2_fwd(const void* act, const void* w2, int a_rows, int max_rows, int m, int h,
                   int num_experts, const int* block_expert, const int* num_m_blocks, void* out,
                   int flags, void* stream) {
  return fc2_fwd_impl(act, w2, a_rows, max_rows, m, h, num_experts, block_expert, num_m_blocks,
                      out, nullptr, flags, stream);
}

// fc2 forward whose output row r is stored at address row_dst[r] (0 = not stored): the EP
// combine's return transfer fused into the GEMM epilogue (rows land in the source rank's
// compact buffer over NVLink).
int moe_gg_fc2_fwd_scatter(const void* act, const void* w2, int a_rows, int max_rows, int m,
                           int h, int num_experts, const int* block_expert,
                           const int* num_m_blocks, const unsigned long long* row_dst, int flags,
                           void* stream) {
  if (!row_dst) return kErrInvalidArg;
  return fc2_fwd_impl(act, w2, a_rows, max_rows, m, h, num_experts, block_expert, num_m_blocks,
                      nullptr, row_dst, flags, stream);
}

// fc2 data-gradient fused with the SwiGLU backward.
//   G[rows, m] = dout[rows, h] * w2_e  (w2[E, h, m] read MN-major)
//   da = G * row_prob (mem-efficient) or G (standard); dprob_partial[row, m/256] = <G, act>
//   d_preact (interleaved like preact) = [da * u * s(g)(1+g(1-s(g))), da * silu(g)]
static int fc2_dgrad_impl(const void* dout, const void* w2, const void* preact, int a_rows,
                          int max_rows, int h, int m, int num_experts, const int* block_expert,
                          const int* num_m_blocks, const float* row_prob, void* d_preact,
                          float* dprob_partial, int flags, const SourceWait* w,
                          void* stream) {
  const int pair = flags & kFlagPair;
  const int split = (flags & kFlagSplit) && pair;
  if (h % BK || m % BN || max_rows % (BM * (pair && !split ? 2 : 1)) || a_rows > max_rows ||
      (split && w))
    return kErrInvalidArg;
  Params p{};
  set_wait(p, w);
  p.num_m_blocks = num_m_blocks;
  p.block_expert = block_expert;
  p.max_m_blocks = max_rows / BM;
  p.num_experts = num_experts;
  p.N = m;
  p.K = h;
  p.out = d_preact;
  p.ldo = 2 * m;
  p.aux = static_cast<const __nv_bfloat16*>(preact);
  p.ld_aux = 2 * m;
  p.row_scale = row_prob;
  p.row_partial = dprob_partial;
  p.ld_partial = (m / BN) * DSW_HALVES;  // one partial per (n-tile, epilogue half)
  return run<false, true, false, EPI_DSWIGLU>(dout, h, a_rows, w2, m, (uint64_t)num_experts * h,
                                              p, p.max_m_blocks, pair,
                                              static_cast<cudaStream_t>(stream), split);
}

int moe_gg_dprob_partials(int m) { return (m / BN) * DSW_HALVES; }

int moe_gg_fc2_dgrad(const void* dout, const void* w2, const void* preact, int a_rows,
                     int max_rows, int h, int m, int num_experts, const int* block_expert,
                     const int* num_m_blocks, const float* row_prob, void* d_preact,
                     float* dprob_partial, int flags, void* stream) {
  return fc2_dgrad_impl(dout, w2, preact, a_rows, max_rows, h, m, num_experts, block_expert,
                        num_m_blocks, row_prob, d_preact, dprob_partial, flags, nullptr, stream);
}

// fc2 data-gradient overlapped with the EP dO dispatch (see moe_gg_fc1_fwd_ep).
int moe_gg_fc2_dgrad_ep(const void* dout, const void* w2, const void* preact, int a_rows,
                        int max_rows, int h, int m, int num_experts, const int* block_expert,
                        const int* num_m_blocks, const float* row_prob, void* d_preact,
                        float* dprob_partial, int flags, const unsigned int* src_flag,
                        const unsigned int* epoch, const unsigned int* block_need,
                        const int* unit_order, int* status, void* stream) {
  if (!src_flag || !epoch || !block_need) return kErrInvalidArg;
  const SourceWait w{src_flag, epoch, block_need, unit_order, status};
  return fc2_dgrad_impl(dout, w2, preact, a_rows, max_rows, h, m, num_experts, block_expert,
                        num_m_blocks, row_prob, d_preact, dprob_partial, flags, &w, stream);
}

static int fc1_dgrad_impl(const void* d_preact, const void* w1, int a_rows, int max_rows,
                          int m, int h, int num_experts, const int* block_expert,
                          const int* num_m_blocks, void* dxp,
                          const unsigned long long* row_dst, int flags, void* stream) {
  const int pair = flags & kFlagPair;
  const int split = (flags & kFlagSplit) && pair;
  if ((2 * m) % BK || h % BN || max_rows % (BM * (pair && !split ? 2 : 1)) || a_rows > max_rows)
    return kErrInvalidArg;
  Params p{};
  p.row_dst = row_dst;
  p.num_m_blocks = num_m_blocks;
  p.block_expert = block_expert;
  p.max_m_blocks = max_rows / BM;
  p.num_experts = num_experts;
  p.N = h;
  p.K = 2 * m;
  p.out = dxp;
  p.ldo = h;
  return run<false, true, false, EPI_BF16>(d_preact, 2 * m, a_rows, w1, h,
                                           (uint64_t)num_experts * 2 * m, p, p.max_m_blocks,
                                           pair, static_cast<cudaStream_t>(stream), split);
}

// fc1 data-gradient: dxp[rows, h] = d_preact[rows, 2m] * w1_e  (w1[E, 2m, h] read MN-major).
int moe_gg_fc1_dgrad(const void* d_preact, const void* w1, int a_rows, int max_rows, int m,
                     int h, int num_experts, const int* block_expert, const int* num_m_blocks,
                     void* dxp, int flags, void* stream) {
  return fc1_dgrad_impl(d_preact, w1, a_rows, max_rows, m, h, num_experts, block_expert,
                        num_m_blocks, dxp, nullptr, flags, stream);
}

// fc1 data-gradient with the dX return transfer fused into the epilogue (see
// moe_gg_fc2_fwd_scatter).
int moe_gg_fc1_dgrad_scatter(const void* d_preact, const void* w1, int a_rows, int max_rows,
                             int m, int h, int num_experts, const int* block_expert,
                             const int* num_m_blocks, const unsigned long long* row_dst,
                             int flags, void* stream) {
  if (!row_dst) return kErrInvalidArg;
  return fc1_dgrad_impl(d_preact, w1, a_rows, max_rows, m, h, num_experts, block_expert,
                        num_m_blocks, nullptr, row_dst, flags, stream);
}

// Weight gradient with the reduction over each expert's token rows:
//   dw[e, M, N] = sum_{r in [off[e], off[e+1])} a[r, 0:M]^T b[r, 0:N]
// a[rows, M], b[rows, N] row-major (read MN-major); off[] multiples of 64; rows >= max_rows
// read as zero. Uses the CTA-pair engine whenever M % 256 == 0.
int moe_gg_wgrad(const void* a, const void* b, int max_rows, int M, int N, int num_experts,
                 const int* expert_offsets, void* dw, void* stream) {
  return moe_gg_wgrad_ex(a, b, max_rows, M, N, num_experts, expert_offsets, dw, 0, stream);
}

// moe_gg_wgrad with flags: bit 0 = programmatic dependent launch. The caller asserts the
// weight gradient does not read what the previous launch on the stream writes (e.g. dW2
// after the fc2 data-gradient: both only read d_O), so it may take the SMs that launch's
// last wave leaves idle; it completes after that launch.
int moe_gg_wgrad_ex(const void* a, const void* b, int max_rows, int M, int N, int num_experts,
                    const int* expert_offsets, void* dw, int flags, void* stream) {
  if (M % BM || N % BN) return kErrInvalidArg;
  Params p{};
  p.expert_offsets = expert_offsets;
  p.num_experts = num_experts;
  p.M = M;
  p.N = N;
  p.out = dw;
  p.ldo = N;
  p.out_expert_stride = (long long)M * N;
  static int force_single = -1;  // MOE_B200_WGRAD_PAIR=0: the 1-CTA engine (A/B)
  if (force_single < 0) {
    const char* e = getenv("MOE_B200_WGRAD_PAIR");
    force_single = (e && e[0] == '0') ? 1 : 0;
  }
  const int pair = !force_single && (M % (2 * BM)) == 0;
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = getenv("MOE_B200_DEBUG_SKIP");
      dbg = e ? atoi(e) : 0;
    }
    p.debug_skip = dbg;
  }
  return run<true, true, true, EPI_BF16>(a, M, max_rows, b, N, max_rows, p,
                                         num_experts * (M / BM), pair,
                                         static_cast<cudaStream_t>(stream), 0, flags & 1);
}

// Same as moe_gg_wgrad with fp32 output (split-K partials of the router weight gradient:
// "experts" are token chunks).
int moe_gg_wgrad_f32(const void* a, const void* b, int max_rows, int M, int N, int num_groups,
                     const int* offsets, float* dw, void* stream) {
  if (M % BM || N % BN) return kErrInvalidArg;
  Params p{};
  p.expert_offsets = offsets;
  p.num_experts = num_groups;
  p.M = M;
  p.N = N;
  p.out = dw;
  p.ldo = N;
  p.out_expert_stride = (long long)M * N;
  const int pair = (M % (2 * BM)) == 0;
  return run<true, true, true, EPI_F32>(a, M, max_rows, b, N, max_rows, p,
                                        num_groups * (M / BM), pair,
                                        static_cast<cudaStream_t>(stream));
}

// Plain grouped-M GEMM with fp32 output (router logits / tests): out[rows, N] = a * b_e^T.
// a_rows: physical rows of a (TMA bound); max_rows: rows of out (multiple of 128).
int moe_gg_gemm_f32(const void* a, const void* b, int a_rows, int max_rows, int K, int N,
                    int num_experts, const int* block_expert, const int* num_m_blocks, float* out,
                    void* stream) {
  if (K % BK || N % BN || max_rows % BM || a_rows > max_rows) return kErrInvalidArg;
  Params p{};
  p.num_m_blocks = num_m_blocks;
  p.block_expert = block_expert;
  p.max_m_blocks = max_rows / BM;
  p.num_experts = num_experts;
  p.N = N;
  p.K = K;
  p.out = out;
  p.ldo = N;
  return run<false, false, false, EPI_F32>(a, K, a_rows, b, K, (uint64_t)num_experts * N, p,
                                           p.max_m_blocks, 0, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
