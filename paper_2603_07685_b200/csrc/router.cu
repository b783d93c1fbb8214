// Router: score function + top-k selection + load-balancing statistics (warp per token),
// and its backward (score Jacobian). The logits GEMM itself runs on the tcgen05 grouped
// GEMM (moe_gg_gemm_f32 with W_r^T padded to 256 rows), see paper_2603_07685_b200/router.py.
//
// Oracle: reference pkg/src/moelab/routing.py
//   route        :71-108  (softmax :85-88, sigma/sum-sigma :89-91, bias on SCORES :95,
//                          stable top-k lowest-index ties :96-101, probs not renormalised
//                          :102, counts :106)
//   aux_loss     :111-120 (coeff * E * sum_i f_i P_i, f = counts / (T*K))
//   gradients    SURVEY Appendix C (score Jacobians; aux term with f constant).
//
// Selection keys are the oracle's fp64 scores (routing.py:85-95): exp(l - max) for softmax
// (the common 1/sum factor is monotone and dropped), sigma(l) = 1/(1+exp(-l)) for
// sigma/sum-sigma, computed in double from the fp32 logits the oracle is given, plus the
// selection bias when present. Distinct fp32 logits give distinct keys except where the fp64
// scores themselves collide (sigmoid saturation to 1.0 from l ~ 34, exp underflow), and
// there the oracle's stable argsort picks the lower expert index, as `better` does; this is
// what makes the indices bit-exact. Non-finite keys (NaN / inf logits: status bit 0, route()
// raises the reference's ValueError) are mapped to -inf so every token still selects K
// valid experts and no index leaves [0, E).
#include "common.cuh"

namespace moe {
namespace router {

constexpr int WARPS = 8;

struct Cand {
  double v;
  int i;
};
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  return a.v > b.v || (a.v == b.v && a.i < b.i);
}

// One token on one warp: scores, selection, outputs. l[j] = logit of expert j*32+lane
// (-inf beyond E). Accumulates the token's scores into part[] and its selections into the
// block's s_counts; sets bad on a non-finite logit.
template <int EPL>
__device__ __forceinline__ void route_token(const float (&l)[EPL], long long t, int E, int K,
                                            int score_fn, const float* __restrict__ sel_bias,
                                            int* __restrict__ topk_idx,
                                            float* __restrict__ topk_prob,
                                            float* __restrict__ topk_score_out, int* s_counts,
                                            float (&part)[EPL], bool& bad) {
  const int lane = lane_id();
  float s[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j)
    if (j * 32 + lane < E && !isfinite(l[j])) bad = true;
  // scores (routing.py:85-91)
  if (score_fn == 0) {
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < EPL; ++j) mx = fmaxf(mx, l[j]);
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      s[j] = (j * 32 + lane < E) ? expf(l[j] - mx) : 0.f;
      sum += s[j];
    }
    sum = warp_sum(sum);
    const float inv = 1.0f / sum;
#pragma unroll
    for (int j = 0; j < EPL; ++j) s[j] *= inv;
  } else {
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      s[j] = (j * 32 + lane < E) ? 1.0f / (1.0f + expf(-l[j])) : 0.f;
      sum += s[j];
    }
    sum = warp_sum(sum);
    const float inv = 1.0f / sum;
#pragma unroll
    for (int j = 0; j < EPL; ++j) s[j] *= inv;
  }
#pragma unroll
  for (int j = 0; j < EPL; ++j) part[j] += s[j];

  // selection key (routing.py:95-97): the fp64 score (up to the common positive factor
  // 1/sum), + bias on the normalised score when a bias is given
  double key[EPL];
  double kmx = -INFINITY, ksum = 0.0;
  if (score_fn == 0) {
#pragma unroll
    for (int j = 0; j < EPL; ++j) kmx = fmax(kmx, (double)l[j]);
    kmx = warp_max_d(kmx);
  }
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = j * 32 + lane;
    double k64 = -INFINITY;
    if (e < E) {
      const double ld = (double)l[j];
      k64 = score_fn == 0 ? exp(ld - kmx) : 1.0 / (1.0 + exp(-ld));
      ksum += k64;
    }
    key[j] = k64;
  }
  if (sel_bias) {
    ksum = warp_sum_d(ksum);
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      if (e < E) key[j] = key[j] / ksum + (double)__ldg(sel_bias + e);
    }
  }
#pragma unroll
  for (int j = 0; j < EPL; ++j)
    if (isnan(key[j])) key[j] = -INFINITY;
  unsigned taken = 0u;  // bit j: expert j*32+lane already selected
  int my_sel = -1;      // lane k keeps the k-th winner
  for (int k = 0; k < K; ++k) {
    Cand c{-INFINITY, 0x7fffffff};  // loses to any real expert, even one keyed -inf
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      if (e < E && !(taken & (1u << j))) {
        Cand o{key[j], e};
        if (better(o, c)) c = o;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      Cand o{__shfl_xor_sync(0xffffffffu, c.v, off), __shfl_xor_sync(0xffffffffu, c.i, off)};
      if (better(o, c)) c = o;
    }
    if (c.i >= E) break;  // unreachable (K <= E leaves a candidate); keeps indices valid
    if ((c.i & 31) == lane) taken |= 1u << (c.i >> 5);
    if (lane == k) my_sel = c.i;
  }
  // write winners ascending by expert index (deterministic combine order)
  int rank = 0;
  for (int k = 0; k < K; ++k) {
    const int o = __shfl_sync(0xffffffffu, my_sel, k);
    if (lane < K && o < my_sel) ++rank;
  }
  float sel_score = 0.f;
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    // score of expert my_sel lives on lane my_sel & 31, slot my_sel >> 5
    const float v = __shfl_sync(0xffffffffu, s[j], my_sel < 0 ? 0 : (my_sel & 31));
    if (my_sel >= 0 && (my_sel >> 5) == j) sel_score = v;
  }
  if (lane < K && my_sel >= 0 && my_sel < E) {
    topk_idx[t * K + rank] = my_sel;
    topk_prob[t * K + rank] = sel_score;
    atomicAdd(&s_counts[my_sel], 1);
  }
  if (topk_score_out) {
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      if (e < E) topk_score_out[t * E + e] = s[j];
    }
  }
}

// Block epilogue shared by both top-k kernels: per-block score column sums (fixed order)
// and the block's counts added to the global counts.
template <int EPL>
__device__ __forceinline__ void flush_block_stats(const float (&part)[EPL], bool bad, int E,
                                                  float (*s_part)[EPL * 32], int* s_counts,
                                                  int* __restrict__ counts,
                                                  float* __restrict__ score_partials,
                                                  int* __restrict__ status) {
  const int warp = warp_id(), lane = lane_id();
  if (bad) atomicOr(status, 1);
#pragma unroll
  for (int j = 0; j < EPL; ++j) s_part[warp][j * 32 + lane] = part[j];
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) acc += s_part[w][e];
    score_partials[(long long)blockIdx.x * E + e] = acc;
    if (s_counts[e]) atomicAdd(&counts[e], s_counts[e]);
  }
}

template <int EPL>
__global__ void __launch_bounds__(WARPS * 32) topk_kernel(
    const float* __restrict__ logits, int ld, int T, int E, int K, int score_fn,
    const float* __restrict__ sel_bias, int* __restrict__ topk_idx, float* __restrict__ topk_prob,
    float* __restrict__ topk_score_out, int* __restrict__ counts,
    float* __restrict__ score_partials, int* __restrict__ status) {
  __shared__ int s_counts[EPL * 32];
  __shared__ float s_part[WARPS][EPL * 32];
  const int warp = warp_id(), lane = lane_id();
  for (int i = threadIdx.x; i < EPL * 32; i += blockDim.x) s_counts[i] = 0;
  __syncthreads();
  float part[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) part[j] = 0.f;
  bool bad = false;
  const int stride = gridDim.x * WARPS;
  for (int t = blockIdx.x * WARPS + warp; t < T; t += stride) {
    const float* row = logits + (long long)t * ld;
    float l[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      l[j] = e < E ? row[e] : -INFINITY;
    }
    route_token<EPL>(l, t, E, K, score_fn, sel_bias, topk_idx, topk_prob, topk_score_out,
                     s_counts, part, bad);
  }
  flush_block_stats<EPL>(part, bad, E, s_part, s_counts, counts, score_partials, status);
}

// W_r [h, E] (row-major, the reference layout) -> shared W_r^T [E][h]: 16-byte global loads
// (eight (k, e) pairs of one or two k rows), independent so they pipeline, scattered into
// the transposed layout with 2-byte shared stores (consecutive threads: consecutive k).
__device__ __forceinline__ void stage_wt(const __nv_bfloat16* __restrict__ w_r, int h, int E,
                                         __nv_bfloat16* wt) {
  const int n8 = h * E / 8;
  const int4* src = reinterpret_cast<const int4*>(w_r);
#pragma unroll 4
  for (int i = threadIdx.x; i < n8; i += blockDim.x) {
    const int4 v = __ldg(src + i);
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int flat = i * 8 + j;
      wt[(flat % E) * h + flat / E] = b[j];
    }
  }
}

// ---------------------------------------------------------------- small-E fused router
// E <= 32 (Mixtral E = 8): the logits GEMM x[T,h] . W_r[h,E] has ~8 FLOP per byte of x, so it
// runs on the CUDA cores inside the top-k kernel instead of a tensor-core tile padded to 256
// columns: x is read once (the HBM floor of the router), W_r^T sits in shared memory, and each
// warp scores TPW tokens at a time so every shared-memory W load feeds TPW x rows. Logits are
// fp32-accumulated (fixed lane order + butterfly, deterministic) and written [T, E] for the
// backward; selection then proceeds exactly as topk_kernel.
template <int EMAX, int TPW>
__global__ void __launch_bounds__(WARPS * 32) fused_small_kernel(
    const int4* __restrict__ x, int T, int hv, const __nv_bfloat16* __restrict__ w_r, int E,
    int K, int score_fn, const float* __restrict__ sel_bias, float* __restrict__ logits,
    int* __restrict__ topk_idx, float* __restrict__ topk_prob,
    float* __restrict__ topk_score_out, int* __restrict__ counts,
    float* __restrict__ score_partials, int P, int* __restrict__ status) {
  extern __shared__ int4 wt4[];  // W_r^T [E][h] bf16, 16-byte vectors
  __shared__ int s_counts[32];
  __shared__ float s_part[WARPS][32];
  const int warp = warp_id(), lane = lane_id();
  const int h = hv * 8;
  stage_wt(w_r, h, E, reinterpret_cast<__nv_bfloat16*>(wt4));
  for (int i = threadIdx.x; i < 32; i += blockDim.x) s_counts[i] = 0;
  // partial rows this grid does not own are zero (the finalize sums P rows)
  for (int r = gridDim.x + blockIdx.x; r < P; r += gridDim.x)
    for (int e = threadIdx.x; e < E; e += blockDim.x) score_partials[(long long)r * E + e] = 0.f;
  __syncthreads();
  float part[1] = {0.f};
  bool bad = false;
  for (long long t0 = ((long long)blockIdx.x * WARPS + warp) * TPW; t0 < T;
       t0 += (long long)gridDim.x * WARPS * TPW) {
    float acc[TPW][EMAX];
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
      for (int e = 0; e < EMAX; ++e) acc[i][e] = 0.f;
    for (int c = lane; c < hv; c += 32) {
      float xf[TPW][8];
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        int4 v = make_int4(0, 0, 0, 0);
        if (t0 + i < T) v = ld_nc_v4(x + (t0 + i) * hv + c);
        const uint32_t* u = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(u[j]);
          xf[i][2 * j] = f.x;
          xf[i][2 * j + 1] = f.y;
        }
      }
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        if (e >= E) break;
        const int4 wv = wt4[e * hv + c];
        const uint32_t* u = reinterpret_cast<const uint32_t*>(&wv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(u[j]);
#pragma unroll
          for (int i = 0; i < TPW; ++i) {
            acc[i][e] = fmaf(xf[i][2 * j], f.x, acc[i][e]);
            acc[i][e] = fmaf(xf[i][2 * j + 1], f.y, acc[i][e]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const long long t = t0 + i;
      float l[1] = {-INFINITY};
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        const float v = warp_sum(acc[i][e]);
        if (lane == e) l[0] = v;
      }
      if (t >= T) continue;  // (warp-uniform)
      if (lane < E) logits[t * E + lane] = l[0];
      if (lane >= E) l[0] = -INFINITY;
      route_token<1>(l, t, E, K, score_fn, sel_bias, topk_idx, topk_prob, topk_score_out,
                     s_counts, part, bad);
    }
  }
  flush_block_stats<1>(part, bad, E, s_part, s_counts, counts, score_partials, status);
}

// aux = coeff * E * sum_i f_i P_i ;  aux_grad[i] = coeff * E * f_i / T  (dL/ds_ti)
// Thread (s, e) of the 1024-thread block sums score-partial rows b = s, s + S, ... of expert e
// (S = 1024 / E subsets; consecutive threads read consecutive experts of a row: coalesced);
// the S subset sums of each expert are then added in subset order (deterministic).
// tile_counts / tile_status (nullable): per-tile counts [P, E] and non-finite flags [P] of the
// tensor-core router; summed here into counts[E] / OR-ed into *status (no memsets, no global
// atomics in the producing kernel).
__global__ void finalize_kernel(int* __restrict__ counts,
                                const float* __restrict__ score_partials, int P, int T, int K,
                                int E, float coeff, float* __restrict__ aux_out,
                                float* __restrict__ aux_grad, float* __restrict__ mean_scores,
                                const int* __restrict__ tile_counts = nullptr,
                                const int* __restrict__ tile_status = nullptr,
                                int* __restrict__ status = nullptr) {
  __shared__ double sub[1024];
  __shared__ double fp[256];
  __shared__ int isub[1024];
  const int S = blockDim.x / E;
  const int e = threadIdx.x % E, sidx = threadIdx.x / E;
  if (tile_counts) {
    // same subset split as the score partials below: coalesced, then a fixed-order combine
    int c = 0;
    if (sidx < S)
      for (int b = sidx; b < P; b += S) c += tile_counts[(long long)b * E + e];
    isub[threadIdx.x] = c;
    int st = 0;
    for (int b = threadIdx.x; b < P; b += blockDim.x) st |= tile_status[b];
    st = __syncthreads_or(st);
    if (threadIdx.x < E) {
      int tot = 0;
      for (int q = 0; q < S; ++q) tot += isub[q * E + threadIdx.x];
      counts[threadIdx.x] = tot;
    }
    if (threadIdx.x == 0 && status) *status = st;
    __syncthreads();
  }
  double ps = 0.0;
  if (sidx < S)
    for (int b = sidx; b < P; b += S) ps += score_partials[(long long)b * E + e];
  sub[threadIdx.x] = ps;
  __syncthreads();
  if (threadIdx.x < E) {
    double tot_p = 0.0;
    for (int q = 0; q < S; ++q) tot_p += sub[q * E + threadIdx.x];
    const double Pm = tot_p / (double)(T > 0 ? T : 1);
    const double f =
        (double)counts[threadIdx.x] / (double)((long long)T * K > 0 ? (long long)T * K : 1);
    fp[threadIdx.x] = f * Pm;
    if (aux_grad) aux_grad[threadIdx.x] = (float)(coeff * E * f / (double)(T > 0 ? T : 1));
    if (mean_scores) mean_scores[threadIdx.x] = (float)Pm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int i = 0; i < E; ++i) tot += fp[i];
    *aux_out = (float)(coeff * E * tot);
  }
}

// dl = J_score^T ds with ds_te = dprob[t,k] (selected) + aux_grad[e]; written as bf16,
// zero-padded to ldd columns (the operand of the router wgrad / dgrad GEMMs).
// OutT = float: compact fp32 [T, E] (ldd = E), the operand of the small-E CUDA-core
// router gradients below.
template <int EPL, typename OutT>
__global__ void __launch_bounds__(WARPS * 32) bwd_kernel(
    const float* __restrict__ logits, int ld, int T, int E, int K, int score_fn,
    const int* __restrict__ topk_idx, const float* __restrict__ dprob,
    const float* __restrict__ aux_grad, OutT* __restrict__ dlogits, int ldd,
    __nv_bfloat16* __restrict__ dlt = nullptr, int ldt = 0, int npad = 0) {
  const int warp = warp_id(), lane = lane_id();
  const int stride = gridDim.x * WARPS;
  for (int t = blockIdx.x * WARPS + warp; t < T; t += stride) {
    const float* row = logits + (long long)t * ld;
    float l[EPL], s[EPL], ds[EPL], sig[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      l[j] = e < E ? row[e] : -INFINITY;
      ds[j] = (e < E && aux_grad) ? __ldg(aux_grad + e) : 0.f;
    }
    // add dprob at the selected experts
    const int my_k = lane < K ? topk_idx[(long long)t * K + lane] : -1;
    const float my_dp = lane < K ? dprob[(long long)t * K + lane] : 0.f;
    for (int k = 0; k < K; ++k) {
      const int e = __shfl_sync(0xffffffffu, my_k, k);
      const float dp = __shfl_sync(0xffffffffu, my_dp, k);
      if (e >= 0 && (e & 31) == lane) {
#pragma unroll
        for (int j = 0; j < EPL; ++j)
          if ((e >> 5) == j) ds[j] += dp;
      }
    }
    float sum = 0.f;
    if (score_fn == 0) {
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < EPL; ++j) mx = fmaxf(mx, l[j]);
      mx = warp_max(mx);
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        s[j] = (j * 32 + lane < E) ? expf(l[j] - mx) : 0.f;
        sum += s[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        sig[j] = (j * 32 + lane < E) ? 1.0f / (1.0f + expf(-l[j])) : 0.f;
        s[j] = sig[j];
        sum += s[j];
      }
    }
    sum = warp_sum(sum);
    const float inv = 1.0f / sum;
    float inner = 0.f;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      s[j] *= inv;
      inner += ds[j] * s[j];
    }
    inner = warp_sum(inner);
    OutT* out = dlogits ? dlogits + (long long)t * ldd : nullptr;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      float dl;
      if (score_fn == 0)
        dl = s[j] * (ds[j] - inner);
      else
        dl = sig[j] * (1.0f - sig[j]) * inv * (ds[j] - inner);
      if (e < E && out) out[e] = static_cast<OutT>(dl);
      // transposed copy dl^T [npad, ldt] (B operand of the small-N router weight gradient)
      if (e < E && dlt) dlt[(long long)e * ldt + t] = __float2bfloat16_rn(dl);
    }
    if (out)
      for (int e = E + lane; e < ldd; e += 32) out[e] = static_cast<OutT>(0.f);
    if (dlt)
      for (int e = E + lane; e < npad; e += 32) dlt[(long long)e * ldt + t] = __float2bfloat16_rn(0.f);
  }
}

// dW_r partials for E <= 16. Block (cx, g): hidden columns [cx*256, +256) (lane = 8 columns,
// one 16-byte x vector per token) over token group g; its 8 warps take interleaved tokens with
// 4 x loads in flight each, then fold their accumulators into warp 0 through shared memory in
// a fixed order. partials[g][k][e] fp32; reduce_blocks_kernel sums the groups in fixed order.
template <int EMAX>
__global__ void __launch_bounds__(WARPS * 32) wgrad_small_kernel(
    const int4* __restrict__ x, int T, int hv, const float* __restrict__ dl, int E,
    int tokens_per_group, float* __restrict__ partials) {
  __shared__ float red[32][8 * EMAX + 1];
  const int warp = warp_id(), lane = lane_id();
  const int c = blockIdx.x * 32 + lane;
  const long long t0 = (long long)blockIdx.y * tokens_per_group;
  const long long t1 = t0 + tokens_per_group < T ? t0 + tokens_per_group : T;
  float acc[8][EMAX];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int e = 0; e < EMAX; ++e) acc[j][e] = 0.f;
  if (c < hv) {
    for (long long t = t0 + warp; t < t1; t += 4 * WARPS) {
      int4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long tq = t + (long long)q * WARPS;
        v[q] = tq < t1 ? ld_nc_v4(x + tq * hv + c) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long tq = t + (long long)q * WARPS;
        if (tq >= t1) break;
        float d[EMAX];
#pragma unroll
        for (int e = 0; e < EMAX; ++e) d[e] = e < E ? __ldg(dl + tq * E + e) : 0.f;
        const uint32_t* u = reinterpret_cast<const uint32_t*>(&v[q]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(u[j]);
#pragma unroll
          for (int e = 0; e < EMAX; ++e) {
            acc[2 * j][e] = fmaf(f.x, d[e], acc[2 * j][e]);
            acc[2 * j + 1][e] = fmaf(f.y, d[e], acc[2 * j + 1][e]);
          }
        }
      }
    }
  }
  // fixed-order fold of the block's warps into warp 0 (w = 1, 2, ..., WARPS-1)
  for (int w = 1; w < WARPS; ++w) {
    if (warp == w)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < EMAX; ++e) red[lane][j * EMAX + e] = acc[j][e];
    __syncthreads();
    if (warp == 0)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < EMAX; ++e) acc[j][e] += red[lane][j * EMAX + e];
    __syncthreads();
  }
  if (warp == 0 && c < hv) {
    float* o = partials + ((long long)blockIdx.y * hv * 8 + (long long)c * 8) * E;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < EMAX; ++e)
        if (e < E) o[j * E + e] = acc[j][e];
  }
}

__global__ void reduce_blocks_kernel(const float* __restrict__ partials, int G, long long n,
                                     float* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = 0.f;
  for (int b = 0; b < G; ++b) acc += partials[(long long)b * n + i];
  out[i] = acc;
}

// Router dX for E <= 16: dx[t, k] = sum_e dl[t, e] W_r[k, e] (bf16 out), warp per token,
// W_r^T staged in shared memory (conflict-free 16-byte lane reads).
template <int EMAX>
__global__ void __launch_bounds__(WARPS * 32) dx_small_kernel(const float* __restrict__ dl,
                                                              int T, int E,
                                                              const __nv_bfloat16* __restrict__ w_r,
                                                              int hv, int4* __restrict__ out) {
  extern __shared__ int4 wt4[];
  stage_wt(w_r, hv * 8, E, reinterpret_cast<__nv_bfloat16*>(wt4));
  __syncthreads();
  const int warp = warp_id(), lane = lane_id();
  for (long long t = (long long)blockIdx.x * WARPS + warp; t < T;
       t += (long long)gridDim.x * WARPS) {
    const float mine = lane < E ? __ldg(dl + t * E + lane) : 0.f;
    float d[EMAX];
#pragma unroll
    for (int e = 0; e < EMAX; ++e) d[e] = __shfl_sync(0xffffffffu, mine, e);
    for (int c = lane; c < hv; c += 32) {
      float a[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = 0.f;
#pragma unroll
      for (int e = 0; e < EMAX; ++e) {
        if (e >= E) break;
        const int4 wv = wt4[e * hv + c];
        const uint32_t* u = reinterpret_cast<const uint32_t*>(&wv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(u[j]);
          a[2 * j] = fmaf(d[e], f.x, a[2 * j]);
          a[2 * j + 1] = fmaf(d[e], f.y, a[2 * j + 1]);
        }
      }
      int4 o;
      o.x = pack_bf16x2(a[0], a[1]);
      o.y = pack_bf16x2(a[2], a[3]);
      o.z = pack_bf16x2(a[4], a[5]);
      o.w = pack_bf16x2(a[6], a[7]);
      st_na_v4(out + t * hv + c, o);
    }
  }
}

static int sms() { return device_sms(); }

}  // namespace router
}  // namespace moe

using namespace moe;
using namespace moe::router;

extern "C" {

// Number of score partial rows the top-k kernel writes for T tokens (workspace query).
int moe_router_num_partials(int T) {
  int blocks = ceil_div_i(T > 0 ? T : 1, WARPS);
  const int cap = 4 * sms();
  return blocks < cap ? blocks : cap;
}

// Score + top-k + counts + per-block score column sums.
//   logits[T, ld] fp32; sel_bias[E] or NULL; score_fn 0 = softmax, 1 = sigmoid.
//   topk_idx[T,K] int32 ascending expert; topk_prob[T,K] fp32 (unbiased score);
//   scores_out[T,E] fp32 or NULL; counts[E] int32 (zeroed here);
//   score_partials[moe_router_num_partials(T), E]; status[1] int32 (bit 0: non-finite).
int moe_router_topk(const float* logits, int ld, int T, int E, int K, int score_fn,
                    const float* sel_bias, int* topk_idx, float* topk_prob, float* scores_out,
                    int* counts, float* score_partials, int* status, void* stream) {
  if (E < 1 || E > 256 || K < 1 || K > 32 || ld < E) return kErrInvalidArg;
  if (K > E) return kErrTopK;
  auto st = static_cast<cudaStream_t>(stream);
  MOE_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(int) * E, st));
  MOE_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(int), st));
  if (T == 0) return kOk;
  const int P = moe_router_num_partials(T);
  const int epl = E <= 32 ? 1 : E <= 64 ? 2 : E <= 128 ? 4 : 8;
#define LAUNCH_TOPK(N)                                                                      \
  topk_kernel<N><<<P, WARPS * 32, 0, st>>>(logits, ld, T, E, K, score_fn, sel_bias, topk_idx, \
                                           topk_prob, scores_out, counts, score_partials,    \
                                           status)
  switch (epl) {
    case 1: LAUNCH_TOPK(1); break;
    case 2: LAUNCH_TOPK(2); break;
    case 4: LAUNCH_TOPK(4); break;
    default: LAUNCH_TOPK(8); break;
  }
#undef LAUNCH_TOPK
  MOE_LAUNCH_CHECK();
  return kOk;
}

// aux loss (device scalar), per-expert aux score-gradient and mean scores.
int moe_router_finalize(const int* counts, const float* score_partials, int T, int K, int E,
                        float coeff, float* aux_out, float* aux_grad, float* mean_scores,
                        void* stream) {
  const int P = moe_router_num_partials(T);
  finalize_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(
      const_cast<int*>(counts), score_partials, T == 0 ? 0 : P, T, K, E, coeff, aux_out,
      aux_grad, mean_scores);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// moe_router_finalize over P explicit score-partial rows (the small-N tensor-core router
// writes one row per 128-token tile).
int moe_router_finalize_p(const int* counts, const float* score_partials, int P, int T, int K,
                          int E, float coeff, float* aux_out, float* aux_grad,
                          float* mean_scores, void* stream) {
  if (E < 1 || E > 256) return kErrInvalidArg;
  finalize_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(
      const_cast<int*>(counts), score_partials, T == 0 ? 0 : P, T, K, E, coeff, aux_out,
      aux_grad, mean_scores);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// moe_router_finalize_p with per-tile counts [P, E] and status flags [P] (summed / OR-ed into
// counts[E] and status[1]).
int moe_router_finalize_tiles(const int* tile_counts, const int* tile_status,
                              const float* score_partials, int P, int T, int K, int E,
                              float coeff, int* counts, int* status, float* aux_out,
                              float* aux_grad, float* mean_scores, void* stream) {
  if (E < 1 || E > 256) return kErrInvalidArg;
  finalize_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(
      counts, score_partials, T == 0 ? 0 : P, T, K, E, coeff, aux_out, aux_grad, mean_scores,
      tile_counts, tile_status, status);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Router backward for the small-N tensor-core router: dl written row-major bf16 [T, ldd]
// (zero beyond E; the dX GEMM's A operand, ldd a multiple of 64) and/or transposed bf16
// dlt[npad, ldt] (rows >= E zero; the weight-gradient B operand). Either may be NULL.
int moe_router_bwd2(const float* logits, int ld, int T, int E, int K, int score_fn,
                    const int* topk_idx, const float* dprob, const float* aux_grad,
                    void* dlogits, int ldd, void* dlt, int ldt, int npad, void* stream) {
  if (E < 1 || E > 256 || K > 32 || (dlogits && ldd < E) || (dlt && (ldt < T || npad < E)))
    return kErrInvalidArg;
  if (T == 0) return kOk;
  // one token per warp: the per-token chain (logits load, max, exp, sum, Jacobian) is
  // latency-bound, so every token gets its own warp (T / 8 blocks, no partial-row cap)
  const int blocks = ceil_div_i(T, WARPS);
  auto st = static_cast<cudaStream_t>(stream);
  auto out = static_cast<__nv_bfloat16*>(dlogits);
  auto ot = static_cast<__nv_bfloat16*>(dlt);
  const int epl = E <= 32 ? 1 : E <= 64 ? 2 : E <= 128 ? 4 : 8;
#define LAUNCH_BWD2(N)                                                                       \
  bwd_kernel<N, __nv_bfloat16><<<blocks, WARPS * 32, 0, st>>>(                               \
      logits, ld, T, E, K, score_fn, topk_idx, dprob, aux_grad, out, ldd, ot, ldt, npad)
  switch (epl) {
    case 1: LAUNCH_BWD2(1); break;
    case 2: LAUNCH_BWD2(2); break;
    case 4: LAUNCH_BWD2(4); break;
    default: LAUNCH_BWD2(8); break;
  }
#undef LAUNCH_BWD2
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Router backward: dlogits[T, ldd] bf16 (zero beyond E).
int moe_router_bwd(const float* logits, int ld, int T, int E, int K, int score_fn,
                   const int* topk_idx, const float* dprob, const float* aux_grad,
                   void* dlogits, int ldd, void* stream) {
  if (E < 1 || E > 256 || K > 32 || ldd < E) return kErrInvalidArg;
  if (T == 0) return kOk;
  const int blocks = moe_router_num_partials(T);
  auto st = static_cast<cudaStream_t>(stream);
  auto out = static_cast<__nv_bfloat16*>(dlogits);
  const int epl = E <= 32 ? 1 : E <= 64 ? 2 : E <= 128 ? 4 : 8;
#define LAUNCH_BWD(N) \
  bwd_kernel<N, __nv_bfloat16><<<blocks, WARPS * 32, 0, st>>>(logits, ld, T, E, K, score_fn,    \
                                                             topk_idx, dprob, aux_grad, out, ldd)
  switch (epl) {
    case 1: LAUNCH_BWD(1); break;
    case 2: LAUNCH_BWD(2); break;
    case 4: LAUNCH_BWD(4); break;
    default: LAUNCH_BWD(8); break;
  }
#undef LAUNCH_BWD
  MOE_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------- small-E fused router
// Eligible when E <= 16, h % 8 == 0 and W_r^T fits the shared-memory budget (E*h*2 bytes);
// larger E uses moe_gg_gemm_f32 + moe_router_topk (the logits GEMM is then tensor-core work).
int moe_router_small_ok(int E, int h) {
  return E >= 1 && E <= 16 && h > 0 && h % 8 == 0 && (long long)E * h * 2 <= 160 * 1024;
}

// route() with the logits computed in-kernel: x[T,h] bf16, w_r[h,E] bf16 (reference layout)
// -> logits[T,E] fp32 and the same outputs as moe_router_topk (score_partials sized by
// moe_router_num_partials(T)).
int moe_router_fused(const void* x, int T, int h, const void* w_r, int E, int K, int score_fn,
                     const float* sel_bias, float* logits, int* topk_idx, float* topk_prob,
                     float* scores_out, int* counts, float* score_partials, int* status,
                     void* stream) {
  if (!moe_router_small_ok(E, h) || K < 1) return kErrInvalidArg;
  if (K > E) return kErrTopK;
  auto st = static_cast<cudaStream_t>(stream);
  MOE_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(int) * E, st));
  MOE_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(int), st));
  if (T == 0) return kOk;
  const int P = moe_router_num_partials(T);
  const int smem = E * h * 2;
  const auto* xv = static_cast<const int4*>(x);
  const auto* w = static_cast<const __nv_bfloat16*>(w_r);
#define LAUNCH_FUSED(EM, TP)                                                                   \
  do {                                                                                         \
    auto kern = fused_small_kernel<EM, TP>;                                                    \
    MOE_CUDA_CHECK(ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem));                \
    int g = ceil_div_i(T, WARPS * TP);                                                         \
    g = g < P ? g : P;                                                                         \
    g = g < 2 * sms() ? g : 2 * sms();                                                         \
    kern<<<g, WARPS * 32, smem, st>>>(xv, T, h / 8, w, E, K, score_fn, sel_bias, logits,       \
                                      topk_idx, topk_prob, scores_out, counts, score_partials, \
                                      P, status);                                              \
  } while (0)
  if (E <= 8)
    LAUNCH_FUSED(8, 8);
  else
    LAUNCH_FUSED(16, 4);
#undef LAUNCH_FUSED
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Router backward, compact fp32 dlogits[T, E] (the small-E gradients' operand).
int moe_router_bwd_f32(const float* logits, int ld, int T, int E, int K, int score_fn,
                       const int* topk_idx, const float* dprob, const float* aux_grad,
                       float* dlogits, void* stream) {
  if (E < 1 || E > 32 || K > 32 || ld < E) return kErrInvalidArg;
  if (T == 0) return kOk;
  bwd_kernel<1, float><<<moe_router_num_partials(T), WARPS * 32, 0,
                         static_cast<cudaStream_t>(stream)>>>(logits, ld, T, E, K, score_fn,
                                                              topk_idx, dprob, aux_grad, dlogits,
                                                              E);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Token groups of moe_router_wgrad_small: enough blocks (x column chunks x groups) for
// ~4 resident blocks per SM.
static int wgrad_small_groups(int T, int h) {
  const int cx = ceil_div_i(h / 8, 32);
  int g = ceil_div_i(4 * sms(), cx);
  const int by_tokens = ceil_div_i(T > 0 ? T : 1, 4 * WARPS);
  return g < by_tokens ? g : by_tokens;
}

// Workspace floats of moe_router_wgrad_small (group partials [G, h, E]).
long long moe_router_wgrad_small_ws(int T, int h, int E) {
  return (long long)wgrad_small_groups(T, h) * h * E;
}

// dW_r[h, E] fp32 = x^T dl for E <= 16 (x read once; fixed-order reductions).
int moe_router_wgrad_small(const void* x, int T, int h, const float* dl, int E, float* ws,
                           float* dw, void* stream) {
  if (E < 1 || E > 16 || h % 8) return kErrInvalidArg;
  auto st = static_cast<cudaStream_t>(stream);
  const long long n = (long long)h * E;
  if (T == 0) {
    MOE_CUDA_CHECK(cudaMemsetAsync(dw, 0, sizeof(float) * n, st));
    return kOk;
  }
  const int G = wgrad_small_groups(T, h);
  const int tpg = ceil_div_i(T, G);
  const dim3 grid(ceil_div_i(h / 8, 32), G);
  const auto* xv = static_cast<const int4*>(x);
  if (E <= 8)
    wgrad_small_kernel<8><<<grid, WARPS * 32, 0, st>>>(xv, T, h / 8, dl, E, tpg, ws);
  else
    wgrad_small_kernel<16><<<grid, WARPS * 32, 0, st>>>(xv, T, h / 8, dl, E, tpg, ws);
  MOE_LAUNCH_CHECK();
  reduce_blocks_kernel<<<(int)ceil_div_ll(n, 256), 256, 0, st>>>(ws, G, n, dw);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Router dX[T, h] bf16 = dl[T, E] . W_r^T for E <= 16 (w_r [h, E] bf16).
int moe_router_dx_small(const float* dl, int T, int E, const void* w_r, int h, void* dx,
                        void* stream) {
  if (!moe_router_small_ok(E, h)) return kErrInvalidArg;
  if (T == 0) return kOk;
  auto st = static_cast<cudaStream_t>(stream);
  const int smem = E * h * 2;
  const int g = ceil_div_i(T, WARPS) < 2 * sms() ? ceil_div_i(T, WARPS) : 2 * sms();
  const auto* w = static_cast<const __nv_bfloat16*>(w_r);
  if (E <= 8) {
    MOE_CUDA_CHECK(ensure_dyn_smem(reinterpret_cast<const void*>(dx_small_kernel<8>), smem));
    dx_small_kernel<8><<<g, WARPS * 32, smem, st>>>(dl, T, E, w, h / 8, static_cast<int4*>(dx));
  } else {
    MOE_CUDA_CHECK(ensure_dyn_smem(reinterpret_cast<const void*>(dx_small_kernel<16>), smem));
    dx_small_kernel<16><<<g, WARPS * 32, smem, st>>>(dl, T, E, w, h / 8,
                                                     static_cast<int4*>(dx));
  }
  MOE_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"
