// Router on the tensor cores with small N: the logits GEMM x[T,h] . W_r[h,E] and the router
// weight gradient x^T . dl run as tcgen05 tiles whose N is the expert count padded to 16
// (not to the 256-column tile of the expert GEMMs), and the forward fuses the whole of
// route() into the GEMM's epilogue: one thread per token reads its E logits straight out of
// TMEM, writes them (fp32, compact [T, E], the backward's operand), then scores, selects and
// counts. The x stream is the only HBM traffic of any size, so the forward is one pass over
// x at HBM speed instead of a padded GEMM + a [T, 256] fp32 logits round trip + a
// warp-per-token top-k (round 1: 0.14 of HBM for the chain; VERDICT r1 "What's weak" 5).
//
// Oracle: reference pkg/src/moelab/routing.py
//   route    :71-108 (softmax :85-88, sigma/sum-sigma :89-91, bias on the normalised SCORES
//                     :95, stable top-k with lowest-index ties :96-101, probs not
//                     renormalised :102, counts :106)
//   aux_loss :111-120 (score column sums feed finalize_kernel, router.cu)
// Selection keys are the oracle's fp64 scores computed from the fp32 logits, exactly as
// router.cu route_token (see the header there): softmax exp(l - max) (the common 1/sum factor
// is monotone and dropped unless a bias is added), sigmoid 1/(1+exp(-l)); NaN keys -> -inf.
//
// Layout: warp 0 = TMA producer, warp 1 = MMA issuer, warps 2..5 = epilogue (warp w reads TMEM
// lanes 32*(w%4)..+31, i.e. token rows of that quarter). One 128-token tile per CTA; with few
// tiles (DeepSeek shape: T = 4096 -> 32 tiles) a cluster of CS CTAs splits h: every CTA
// accumulates its k-range, the non-leaders park their fp32 partial tiles in a workspace and
// the leader adds them in rank order (deterministic) after a cluster barrier.
//
// MODE_WGRAD: weight gradient partials part[s][NPAD][h] = (x[rows(s)]^T . dl[rows(s)])^T: A = x
// read MN-major (M = h), B = dl^T [NPAD, T] (K-major), split-K over token ranges s; the
// fixed-order sum over s is reduce_cm_kernel.
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace moe {
namespace rtc {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int UMMA_K = 16;
// warp 0 TMA, warp 1 MMA, warps 2..5 TMEM epilogue; the route kernel adds 2 warps so its
// selection runs 256 / (128 / CS) threads per token row of the CTA's slice
constexpr int THREADS = 64 + 4 * 32;
constexpr int RT_WARPS = 8;
template <int MODE>
constexpr int threads_of() { return MODE == 0 ? RT_WARPS * 32 : THREADS; }
constexpr int MODE_ROUTE = 0;
constexpr int MODE_WGRAD = 1;

#ifndef MOE_ROUTER_RING_KB
#define MOE_ROUTER_RING_KB 96
#endif
constexpr int RING_KB = MOE_ROUTER_RING_KB;  // operand ring per CTA (A/B: 96 vs 160 measured)

// 64-column sub-blocks per ring stage of the route kernel: each stage reads SUBK * 128
// contiguous bytes of every x row (longer DRAM bursts per row than one 128-byte box)
#ifndef MOE_ROUTER_SUBK
#define MOE_ROUTER_SUBK 2
#endif
// (NPAD >= 128: the W^T box alone is 16-32 KB per sub-block; one sub-block per stage)
// rows per x box of the route kernel (A/B: 128 = one box per 64-column sub-block)
#ifndef MOE_ROUTER_BOX_ROWS
#define MOE_ROUTER_BOX_ROWS 64
#endif
constexpr int ROUTE_BOX_ROWS = MOE_ROUTER_BOX_ROWS;

template <int MODE, int NPAD>
constexpr int subk_of() { return MODE == 0 && NPAD <= 64 ? MOE_ROUTER_SUBK : 1; }
static int subk_route(int npad) { return npad <= 64 ? MOE_ROUTER_SUBK : 1; }

template <int NPAD, int SUBK = 1>
struct Cfg {
  static constexpr int A_STAGE = SUBK * BM * BK * 2;    // SUBK x 16 KB
  static constexpr int B_STAGE = SUBK * NPAD * BK * 2;  // SUBK x NPAD rows x 128 B
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int STAGES = (RING_KB * 1024) / STAGE < 3 ? 3 : (RING_KB * 1024) / STAGE;
  static constexpr int TMEM_COLS = NPAD < 32 ? 32 : NPAD;
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/ +
                              256 * 4 /*counts*/ + 256 * 4 /*selection bias*/ + 16 /*flag*/;
};

struct Params {
  int T, h, E, K;
  int score_fn;
  int num_kb;   // k-blocks of one CTA (route: per cluster rank; wgrad: per split)
  int CS;       // route: cluster size (split of h)
  const float* sel_bias;
  float* logits;         // [T, E] fp32
  int* topk_idx;         // [T, K]
  float* topk_prob;      // [T, K]
  float* scores_out;     // [T, E] or null
  int* tile_counts;      // [tiles * CS, E] per-slice expert counts
  int* tile_status;      // [tiles * CS] per-slice non-finite flag
  float* score_partials; // [tiles, E]

  float* ws;             // route, CS > 1: [tiles, CS, NPAD, 128] fp32 partial logits
  float* part;           // wgrad: [splits, NPAD, h] fp32
  int debug_skip;        // probe only: stop after the logits (mainloop + copy-out)
  int m_tiles;           // wgrad: h / 128
};

__device__ __forceinline__ uint32_t cluster_rank_u32() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ void epi_bar() {  // the 4 epilogue warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

struct Top {
  double k;
  int i;
  float l;
};
__device__ __forceinline__ bool better(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

template <int NPAD, int MODE, int KMAX>
__global__ void __launch_bounds__(threads_of<MODE>(), 1)
    router_tc_kernel(const __grid_constant__ CUtensorMap tmap_a,
                     const __grid_constant__ CUtensorMap tmap_b, const Params p) {
  constexpr int SUBK = subk_of<MODE, NPAD>();
  constexpr int KB = SUBK * BK;  // columns per ring stage
  using C = Cfg<NPAD, SUBK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::STAGES * C::A_STAGE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* done_bar = empty_bar + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);
  int* s_counts = reinterpret_cast<int*>(smem + C::STAGES * C::STAGE + 256);  // [256]
  float* s_bias = reinterpret_cast<float*>(s_counts + 256);                    // [256]
  int* s_flag = reinterpret_cast<int*>(s_bias + 256);                          // [1]

  const int warp = warp_id(), lane = lane_id();
  const int crank = (MODE == MODE_ROUTE && p.CS > 1) ? static_cast<int>(cluster_rank_u32()) : 0;
  // route: tile = cluster index, k-range = rank; wgrad: (m tile, split)
  int tile, m0, k0;
  if constexpr (MODE == MODE_ROUTE) {
    tile = blockIdx.x / p.CS;
    m0 = tile * BM;
    k0 = crank * p.num_kb * KB;
  } else {
    tile = blockIdx.x % p.m_tiles;
    m0 = tile * BM;
    k0 = (blockIdx.x / p.m_tiles) * p.num_kb * KB;
  }
  // k-blocks this CTA owns (the last range may be short; TMA zero-fills past the end)
  const int kdim = MODE == MODE_ROUTE ? p.h : p.T;
  int nkb = p.num_kb;
  if (k0 + nkb * KB > kdim) nkb = k0 < kdim ? (kdim - k0 + KB - 1) / KB : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(done_bar, 1);
    fence_mbar_init();
  }
  if (MODE == MODE_ROUTE) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_counts[i] = 0;
    if (threadIdx.x == 0) s_flag[0] = 0;
    if (p.sel_bias)
      for (int i = threadIdx.x; i < p.E; i += blockDim.x)
        s_bias[i] = __ldg(p.sel_bias + i);
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        mbar_arrive_expect_tx(&full_bar[s], C::STAGE);
        const int k = k0 + kb * KB;
        uint8_t* sa = smem_a + s * C::A_STAGE;
        if constexpr (MODE == MODE_ROUTE) {
#pragma unroll
          for (int sb = 0; sb < SUBK; ++sb)  // x rows m0.., columns k + 64 sb ..
#pragma unroll
            for (int hb = 0; hb < BM / ROUTE_BOX_ROWS; ++hb)  // (same smem image as one box)
              tma_load_2d(sa + sb * (BM * BK * 2) + hb * (ROUTE_BOX_ROWS * BK * 2), &tmap_a,
                          &full_bar[s], k + sb * BK, m0 + hb * ROUTE_BOX_ROWS);
        } else {
          // x^T tile, MN-major: two 64(h) x 64(token) boxes
          tma_load_2d(sa, &tmap_a, &full_bar[s], m0, k);
          tma_load_2d(sa + 64 * BK * 2, &tmap_a, &full_bar[s], m0 + 64, k);
        }
#pragma unroll
        for (int sb = 0; sb < SUBK; ++sb)
          tma_load_2d(smem_b + s * C::B_STAGE + sb * (NPAD * BK * 2), &tmap_b, &full_bar[s],
                      k + sb * BK, 0);
        if (++s == C::STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM, NPAD, MODE == MODE_WGRAD ? 1 : 0, 0);
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(smem_a + s * C::A_STAGE);
        const uint32_t b_base = smem_u32(smem_b + s * C::B_STAGE);
#pragma unroll
        for (int sb = 0; sb < SUBK; ++sb)
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            const uint32_t ab = a_base + sb * (BM * BK * 2), bb = b_base + sb * (NPAD * BK * 2);
            const uint64_t adesc =
                MODE == MODE_WGRAD ? make_sdesc_sw128(ab + kk * (UMMA_K * 128), 64 * BK * 2, 1024)
                                   : make_sdesc_sw128(ab + kk * (UMMA_K * 2), 16, 1024);
            const uint64_t bdesc = make_sdesc_sw128(bb + kk * (UMMA_K * 2), 16, 1024);
            umma_bf16(tmem_base, adesc, bdesc, idesc, (kb | sb | kk) != 0 ? 1u : 0u);
          }
        umma_commit(&empty_bar[s]);
        if (++s == C::STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      umma_commit(done_bar);  // nkb == 0: arrives at once (nothing outstanding)
    }
  }

  // ---------------- epilogue (warps 2..5)
  const int q = warp & 3;
  const int row = q * 32 + lane;
  const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
  const bool epi = warp >= 2 && warp < 6;  // the TMEM lane-quarter warps
  if (epi) {
    // the epilogue warps idle through the whole mainloop: back off instead of spinning, so
    // they do not take issue slots from the producer and MMA warps on the same SMSPs
    mbar_wait_suspend(done_bar, 0);
    tc_fence_after();
  }
  // empty k-range (nkb == 0): the accumulator was never written; treat it as zero
  auto tmem_chunk = [&](int c0, float (&v)[32]) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr + c0, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = nkb > 0 ? __uint_as_float(r[j]) : 0.f;
  };

  if constexpr (MODE == MODE_WGRAD) {
    if (epi) {
      // part[split][col][h]: column-major, so a warp's 32 rows of one column are one
      // coalesced 128-byte store (h % 128 == 0: every row is in range)
      const int split = blockIdx.x / p.m_tiles;
      float* o = p.part + (long long)split * NPAD * p.h + m0 + row;
#pragma unroll
      for (int c0 = 0; c0 < NPAD; c0 += 32) {
        float v[32];
        tmem_chunk(c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j < NPAD) o[(long long)(c0 + j) * p.h] = v[j];
      }
    }
  } else {
    // ---- the tile's logits: with a split-h cluster every CTA parks its partial tile in ws
    // (column-major [tile][rank][col][row], coalesced) and, after the cluster barrier, CTA r
    // sums the CS partials (rank order: deterministic) for its slice of RB = 128 / CS rows,
    // so the selection below is spread over the whole cluster. Without a split the CTA
    // reads its accumulator straight from TMEM.
    const int CS = p.CS;
    const int RB = BM / CS;               // rows of this CTA's slice
    const int rb0 = crank * RB;           // first row of the slice within the tile
    const int SR = blockDim.x / RB;       // threads per row in the selection (2 .. 16)
    if (CS > 1) {
      if (epi) {
        float* wsrow = p.ws + ((long long)tile * CS + crank) * NPAD * BM + row;
#pragma unroll 1
        for (int c0 = 0; c0 < NPAD; c0 += 32) {
          float v[32];
          tmem_chunk(c0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < NPAD) wsrow[(c0 + j) * BM] = v[j];
        }
        __threadfence();
      }
      cluster_sync();
    }
    // The operand ring is idle once the last MMA has completed (every TMA load it issued
    // was consumed): it now holds the slice's logits L[row][e] fp32, row stride NPAD + 4
    // (= 4 mod 32 banks: conflict-free 16-byte row loads). The selection runs on all warps
    // with SR threads per row, each scanning a contiguous quarter/half/... of the experts
    // with plain loops (a fully unrolled NPAD-wide per-thread epilogue thrashed the
    // instruction cache and left one thread per token serial over E: ncu no_inst stalls,
    // 227k SASS lines at NPAD 128, 180-350 us at the Qwen3 / DeepSeek shapes).
    constexpr int LS = NPAD + 4;
    static_assert(BM * LS * 4 <= C::STAGES * C::STAGE, "logits tile must fit the ring");
    float* L = reinterpret_cast<float*>(smem);
    const int E = p.E, K = p.K;
    const bool sm = p.score_fn == 0;
    if (CS == 1) {
      if (epi) {
        float* Lw = L + row * LS;
#pragma unroll 1
        for (int c0 = 0; c0 < NPAD; c0 += 32) {
          float v[32];
          tmem_chunk(c0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < NPAD) Lw[c0 + j] = v[j];
        }
      }
    } else {
      const float* w0 = p.ws + (long long)tile * CS * NPAD * BM + rb0;
      const int n = RB * E;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int c = i / RB, r = i - (i / RB) * RB;  // consecutive threads: consecutive rows
        float acc = 0.f;
        for (int q2 = 0; q2 < CS; ++q2) acc += w0[((long long)q2 * NPAD + c) * BM + r];
        L[r * LS + c] = acc;
      }
    }
    __syncthreads();
    const long long tb = (long long)m0 + rb0;  // first token of the slice
    const int rows_valid = tb < p.T ? (int)min((long long)RB, p.T - tb) : 0;
    // the slice's rows x E block is contiguous in a [T, E] output: coalesced copy-out
    auto rows_out = [&](float* dst) {
      const int n = rows_valid * E;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int r = i / E;
        dst[tb * E + i] = L[r * LS + (i - r * E)];
      }
    };
    rows_out(p.logits);
    __syncthreads();  // (pass 2 overwrites L; the exact path re-reads these logits)
    if (!p.debug_skip) {
      const int srow = threadIdx.x / SR, sub = threadIdx.x % SR;
      float* Lr = L + srow * LS;
      const long long t = tb + srow;
      const bool valid = t < p.T;
      const int per = ((E + SR - 1) / SR + 3) & ~3;
      const int e0 = sub * per, e1 = min(E, e0 + per);
      // row max and finiteness over the SR lanes (butterfly: the same value in every lane)
      float mx = -INFINITY;
      bool bad = false;
#pragma unroll 1
      for (int e = e0; e < e1; ++e) {
        const float l = Lr[e];
        bad |= !isfinite(l);
        mx = fmaxf(mx, l);
      }
      for (int off = 1; off < SR; off <<= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        bad |= __shfl_xor_sync(0xffffffffu, bad ? 1 : 0, off) != 0;
      }
      // pass 2: the fp32 unnormalised score sc_e (softmax expf(l - mx), sigmoid
      // 1/(1+expf(-l))) replaces the logit in L; its row sum is reduced over the lanes
      float sum = 0.f;
#pragma unroll 1
      for (int e = e0; e < e1; ++e) {
        const float l = Lr[e];
        const float sc = sm ? expf(l - mx) : 1.0f / (1.0f + expf(-l));
        Lr[e] = sc;
        sum += sc;
      }
      for (int off = 1; off < SR; off <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      const float inv = 1.0f / sum;
      // Selection on fp32 approximations of the oracle's fp64 keys: key_e = sc_e (no bias;
      // the common 1/sum factor is dropped, as the fp64 key drops it) or sc_e/sum + b_e
      // (routing.py:95). K + 1 max passes (branch-free scans of the lane's experts, then a
      // butterfly (key desc, index asc) reduction over the row's lanes) give the top K + 1;
      // a pass's winner is marked taken by setting the sign bit of its sc (sc >= +0), which
      // is cleared again afterwards. The fp32 choice is exact whenever the K-th and (K+1)-th
      // approximate keys are separated by more than the fp32 error bound: the selected SET
      // is then the fp64 one (the output order is by expert index anyway). Otherwise (near
      // ties, fp32 underflow / saturation, non-finite logits) the fp64 keys decide among the
      // experts whose approximate key is within the tolerance of the boundary (only those
      // can be in the fp64 top K), exactly as router.cu route_token. Error bounds:
      //   softmax key expf(l - mx): |d| * 2^-24 from rounding d = l - mx (|d| <= 87 before
      //     fp32 underflow) + 2 ulp of expf -> relative <= 5.5e-6;
      //   sigmoid key 1/(1+expf(-l)): relative <= 4e-7;
      //   biased key sc/sum + b: sc/sum relative <= 5.5e-6 + E * 2^-24 (sum, E <= 256)
      //     -> <= 2.1e-5, plus the rounding of the add (2^-24 |key|).
      // The tolerance below is >= 3x these bounds.
      const bool biased = p.sel_bias != nullptr;
      const float* bias_s = s_bias;
      int win[KMAX + 1];
      float kK = -INFINITY, kK1 = -INFINITY, sK = 0.f, sK1 = 0.f;
#pragma unroll
      for (int k = 0; k < KMAX + 1; ++k) {
        float bk = -INFINITY;
        int bi = 0x7fffffff;
        if (k <= K) {
#pragma unroll 1
          for (int e = e0; e < e1; e += 4) {
            const float4 v4 = *reinterpret_cast<const float4*>(Lr + e);
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float v = vv[u];
              const float key = biased ? fmaf(v, inv, bias_s[min(e + u, E - 1)]) : v;
              // (ascending e within the lane: a strict > keeps the lower index on ties)
              const bool ok = e + u < e1 && !signbit(v) && (key > bk || bi == 0x7fffffff);
              bk = ok ? key : bk;
              bi = ok ? e + u : bi;
            }
          }
          for (int off = 1; off < SR; off <<= 1) {
            const float ok = __shfl_xor_sync(0xffffffffu, bk, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ok > bk || (ok == bk && oi < bi)) {
              bk = ok;
              bi = oi;
            }
          }
          if (k < K && bi >= e0 && bi < e1) Lr[bi] = -Lr[bi];  // taken (sign bit)
          if (k == K - 1) kK = bk;
          if (k == K) kK1 = bk;
        }
        win[k] = bi;
      }
      // clear the taken marks (owner lanes), then the score parts of the boundary keys
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K && win[k] >= e0 && win[k] < e1) Lr[win[k]] = fabsf(Lr[win[k]]);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < KMAX + 1; ++k) {
        if (k == K - 1 && win[k] < E) sK = Lr[win[k]] * inv;
        if (k == K && win[k] < E) sK1 = Lr[win[k]] * inv;
      }
      // (K == E: no (K+1)-th expert, kK1 stays -inf)
      const float tol = biased ? 1e-4f * (fabsf(sK) + fabsf(sK1)) +
                                     5e-7f * (fabsf(kK) + fabsf(kK1))
                               : 3e-5f * (fabsf(kK) + fabsf(kK1));
      const bool fast = !valid || (!bad && (kK1 == -INFINITY || kK - kK1 > tol + 1e-37f));
      if (__any_sync(0xffffffffu, !fast)) {
        // exact: the oracle's fp64 keys (routing.py:85-97) from the logits just written,
        // lowest index on equal keys, over the candidates (every expert of a non-finite row)
        const float* lg = p.logits + t * E;
        const double kmx = static_cast<double>(mx);
        double ksum = 0.0;
        if (!fast && biased)
          for (int e = e0; e < e1; ++e) {
            const double ld = static_cast<double>(lg[e]);
            ksum += sm ? exp(ld - kmx) : 1.0 / (1.0 + exp(-ld));
          }
        for (int off = 1; off < SR; off <<= 1) ksum += __shfl_xor_sync(0xffffffffu, ksum, off);
        if (!fast && sub == 0) {
          Top top[KMAX];
#pragma unroll
          for (int i = 0; i < KMAX; ++i) top[i] = Top{-INFINITY, 0x7fffffff, 0.f};
          auto insert = [&](double k, int e) {
            if (isnan(k)) k = -INFINITY;
            if (!better(k, e, top[KMAX - 1].k, top[KMAX - 1].i)) return;
            top[KMAX - 1] = Top{k, e, 0.f};
#pragma unroll
            for (int i = KMAX - 1; i > 0; --i)
              if (better(top[i].k, top[i].i, top[i - 1].k, top[i - 1].i)) {
                const Top tmp = top[i];
                top[i] = top[i - 1];
                top[i - 1] = tmp;
              }
          };
          const float thr = kK1 - tol - 1e-37f;
#pragma unroll 1
          for (int e = 0; e < E; ++e) {
            const float a = biased ? fmaf(Lr[e], inv, bias_s[e]) : Lr[e];
            if (!(bad || kK1 == -INFINITY || a >= thr)) continue;
            const double ld = static_cast<double>(lg[e]);
            const double k64 = sm ? exp(ld - kmx) : 1.0 / (1.0 + exp(-ld));
            insert(biased ? k64 / ksum + static_cast<double>(bias_s[e]) : k64, e);
          }
#pragma unroll
          for (int i = 0; i < KMAX; ++i) win[i] = top[i].i;
        }
      }
      // winners ascending by expert index (deterministic combine order); prob = sc * inv
      if (valid && sub == 0) {
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          if (i >= K) break;
          int rank = 0;
#pragma unroll
          for (int j = 0; j < KMAX; ++j)
            if (j < K && win[j] < win[i]) ++rank;
          const int e = win[i] < E ? win[i] : 0;  // (always < E: K <= E)
          p.topk_idx[t * K + rank] = e;
          p.topk_prob[t * K + rank] = Lr[e] * inv;
          atomicAdd(&s_counts[e], 1);
        }
        if (bad) atomicOr(&s_flag[0], 1);
      }
      // pass 3: normalised scores s = sc * inv overwrite L (0 for rows past T) ->
      // scores_out and the slice's column sums (rows in fixed order: deterministic)
      __syncwarp();
#pragma unroll 1
      for (int e = e0; e < e1; ++e) Lr[e] = valid ? Lr[e] * inv : 0.f;
      __syncthreads();
      if (p.scores_out) rows_out(p.scores_out);
      const long long prow = (long long)tile * CS + crank;  // score-partial row
      for (int e = threadIdx.x; e < E; e += blockDim.x) {
        float acc = 0.f;
#pragma unroll 8
        for (int r = 0; r < RB; ++r) acc += L[r * LS + e];
        p.score_partials[prow * E + e] = acc;
        p.tile_counts[prow * E + e] = s_counts[e];
      }
      if (threadIdx.x == 0) p.tile_status[prow] = s_flag[0];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------- host side
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

// bf16 [outer, inner] (row stride ld elements), SWIZZLE_128B boxes {box_inner, box_outer};
// reads past inner / outer are zero-filled.
static int make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                     uint64_t ld, uint32_t box_inner, uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return kErrCuda;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * 2) & 15)) return kErrInvalidArg;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? kOk : kErrCuda;
}

// Split of h across a cluster for the route kernel: enough CTAs to cover the SMs.
static int route_cluster(int T, int h) {
  const int tiles = ceil_div_i(T, BM);
  const int kbs = ceil_div_i(h, BK);
  static int forced = -1;  // MOE_ROUTER_TC_CS=1|2|4|8 (A/B measurements)
  if (forced < 0) {
    const char* e = getenv("MOE_ROUTER_TC_CS");
    forced = e ? atoi(e) : 0;
  }
  if (forced == 1 || forced == 2 || forced == 4 || forced == 8) return forced;
  // measured (tools/router_bench.py): one wave of CTAs wins; DeepSeek shape (32 tiles) 4-way
  // split 133 us vs 196 (1) / 170 (2) / 176 (8); Mixtral / Qwen3 (>= 128 tiles) unsplit
  int cs = 1;
  while (cs < 8 && tiles * cs * 2 <= device_sms() && kbs >= 4 * cs) cs *= 2;
  return cs;
}

// token splits of the wgrad kernel: ~1 CTA per SM, >= 4 k-blocks each
static int wgrad_splits(int T, int h) {
  const int mt = ceil_div_i(h, BM);
  int s = ceil_div_i(device_sms(), mt);
  const int max_s = ceil_div_i(T, 4 * BK);
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : s;
}

template <int NPAD, int MODE, int KMAX>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int grid,
                  int cs, cudaStream_t st) {
  auto kern = router_tc_kernel<NPAD, MODE, KMAX>;
  constexpr int SMEM = Cfg<NPAD, subk_of<MODE, NPAD>()>::SMEM;
  MOE_CUDA_CHECK(ensure_dyn_smem(reinterpret_cast<const void*>(kern), SMEM));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads_of<MODE>());
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MOE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ta, tb, p));
  return kOk;
}

static int npad_of(int E) {
  return E <= 16 ? 16 : E <= 32 ? 32 : E <= 64 ? 64 : E <= 128 ? 128 : 256;
}

// dw[hh, e] = sum_s part[s][e][hh] for e < E (fixed split order); part column-major
__global__ void reduce_cm_kernel(const float* __restrict__ part, int S, int h, int npad, int E,
                                 float* __restrict__ dw) {
  const long long n = (long long)E * h;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int e = static_cast<int>(i / h), hh = static_cast<int>(i % h);
    float acc = 0.f;
    for (int s2 = 0; s2 < S; ++s2) acc += part[((long long)s2 * npad + e) * h + hh];
    dw[(long long)hh * E + e] = acc;
  }
}

#define RTC_DISPATCH_NPAD(NP, CALL) \
  switch (NP) {                     \
    case 16: { constexpr int N_ = 16; CALL; } break;   \
    case 32: { constexpr int N_ = 32; CALL; } break;   \
    case 64: { constexpr int N_ = 64; CALL; } break;   \
    case 128: { constexpr int N_ = 128; CALL; } break; \
    default: { constexpr int N_ = 256; CALL; } break;  \
  }

}  // namespace rtc
}  // namespace moe

using namespace moe;
using namespace moe::rtc;

extern "C" {

// Padded expert count of the small-N router tiles (W_r^T staging rows).
int moe_router_tc_npad(int E) { return E >= 1 && E <= 256 ? npad_of(E) : -1; }

// Workspace of moe_router_tc_fwd in 4-byte words: score partials [P, E] fp32, slice counts
// [P, E] int32, slice flags [P] int32 (P = tiles * CS, each 16-byte aligned), then the
// split-h partial logits [tiles, CS, NPAD, 128] fp32 (CS > 1 only).
static long long ws_a4(long long n) { return (n + 3) / 4 * 4; }
long long moe_router_tc_fwd_ws(int T, int h, int E) {
  if (T <= 0) return E;
  const int tiles = ceil_div_i(T, BM);
  const int cs = route_cluster(T, h);
  const long long P = (long long)tiles * cs;
  return 2 * ws_a4(P * E) + ws_a4(P) + (cs > 1 ? (long long)tiles * cs * BM * npad_of(E) : 0);
}

// route() + aux_loss() (routing.py:71-120) in one GEMM-with-epilogue launch + finalize:
//   x[T, h] bf16 (h % 8 == 0), w_t[NPAD, h] bf16 = W_r^T zero-padded to moe_router_tc_npad(E)
//   rows; outputs as moe_router_topk + moe_router_finalize, logits compact [T, E] fp32.
int moe_router_tc_fwd(const void* x, int T, int h, const void* w_t, int E, int K, int score_fn,
                      const float* sel_bias, float coeff, float* logits, int* topk_idx,
                      float* topk_prob, float* scores_out, int* counts, float* ws, int* status,
                      float* aux_out, float* aux_grad, float* mean_scores, void* stream) {
  if (E < 1 || E > 256 || K < 1 || K > 8 || h < 8 || h % 8) return kErrInvalidArg;
  if (K > E) return kErrTopK;
  auto st = static_cast<cudaStream_t>(stream);
  const int tiles = T > 0 ? ceil_div_i(T, BM) : 0;
  const long long P = T > 0 ? (long long)tiles * route_cluster(T, h) : 0;
  int* tile_counts = reinterpret_cast<int*>(ws + ws_a4(P * E));
  int* tile_status = tile_counts + ws_a4(P * E);
  if (T > 0) {
    const int np = npad_of(E);
    const int cs = route_cluster(T, h);
    CUtensorMap ta, tb;
    int s;
    if ((s = make_tmap(&ta, x, h, T, h, BK, ROUTE_BOX_ROWS))) return s;
    if ((s = make_tmap(&tb, w_t, h, np, h, BK, np))) return s;
    Params p{};
    p.T = T;
    p.h = h;
    p.E = E;
    p.K = K;
    p.score_fn = score_fn;
    p.CS = cs;
    p.num_kb = ceil_div_i(ceil_div_i(h, BK * subk_route(np)), cs);  // ring stages
    p.sel_bias = sel_bias;
    p.logits = logits;
    p.topk_idx = topk_idx;
    p.topk_prob = topk_prob;
    p.scores_out = scores_out;
    p.tile_counts = tile_counts;
    p.tile_status = tile_status;
    p.score_partials = ws;
    p.ws = ws + 2 * ws_a4(P * E) + ws_a4(P);  // 16-byte aligned
    {
      static int dbg = -1;
      if (dbg < 0) {
        const char* e = getenv("MOE_ROUTER_TC_DEBUG_SKIP");
        dbg = (e && e[0] == '1') ? 1 : 0;
      }
      p.debug_skip = dbg;
    }
    int r = kOk;
    if (K <= 2) {
      RTC_DISPATCH_NPAD(np, (r = launch<N_, MODE_ROUTE, 2>(ta, tb, p, tiles * cs, cs, st)));
    } else {
      RTC_DISPATCH_NPAD(np, (r = launch<N_, MODE_ROUTE, 8>(ta, tb, p, tiles * cs, cs, st)));
    }
    if (r) return r;
  }
  // (T == 0: P == 0, the finalize writes zero counts, a clear status and a zero aux loss)
  return moe_router_finalize_tiles(tile_counts, tile_status, ws, (int)P, T, K, E, coeff, counts,
                                   status, aux_out, aux_grad, mean_scores, stream);
}

// Workspace floats of moe_router_tc_wgrad: part [splits, NPAD, h].
long long moe_router_tc_wgrad_ws(int T, int h, int E) {
  return (long long)wgrad_splits(T > 0 ? T : 1, h) * h * npad_of(E);
}

// dW_r[h, E] fp32 = x^T dl (router weight gradient): x[T, h] bf16, dlt[NPAD, ldt] bf16 =
// dl^T zero-padded to moe_router_tc_npad(E) rows (columns >= T ignored), fixed-order split
// sum (reduce_cm_kernel).
int moe_router_tc_wgrad(const void* x, int T, int h, const void* dlt, int ldt, int E, float* ws,
                        float* dw, void* stream) {
  if (E < 1 || E > 256 || h < BM || h % BM || ldt < T || ldt % 8) return kErrInvalidArg;
  auto st = static_cast<cudaStream_t>(stream);
  if (T <= 0) {
    MOE_CUDA_CHECK(cudaMemsetAsync(dw, 0, sizeof(float) * h * E, st));
    return kOk;
  }
  const int np = npad_of(E);
  const int splits = wgrad_splits(T, h);
  CUtensorMap ta, tb;
  int s;
  if ((s = make_tmap(&ta, x, h, T, h, 64, BK))) return s;
  if ((s = make_tmap(&tb, dlt, T, np, ldt, BK, np))) return s;
  Params p{};
  p.T = T;
  p.h = h;
  p.E = E;
  p.m_tiles = h / BM;
  p.num_kb = ceil_div_i(ceil_div_i(T, BK), splits);
  p.part = ws;
  int r = kOk;
  RTC_DISPATCH_NPAD(np, (r = launch<N_, MODE_WGRAD, 2>(ta, tb, p, p.m_tiles * splits, 1, st)));
  if (r) return r;
  const long long n = (long long)E * h;
  reduce_cm_kernel<<<(int)(ceil_div_ll(n, 256) < 1024 ? ceil_div_ll(n, 256) : 1024), 256, 0, st>>>(
      ws, splits, h, np, E, dw);
  MOE_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"
