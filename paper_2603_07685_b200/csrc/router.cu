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
    float l[EPL], s[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      l[j] = e < E ? row[e] : -INFINITY;
      if (e < E && !isfinite(l[j])) bad = true;
    }
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
      const int e = j * 32 + lane;
      // score of expert my_sel lives on lane my_sel & 31, slot my_sel >> 5
      const float v = __shfl_sync(0xffffffffu, s[j], my_sel < 0 ? 0 : (my_sel & 31));
      if (my_sel >= 0 && (my_sel >> 5) == j) sel_score = v;
      (void)e;
    }
    if (lane < K && my_sel >= 0 && my_sel < E) {
      topk_idx[(long long)t * K + rank] = my_sel;
      topk_prob[(long long)t * K + rank] = sel_score;
      atomicAdd(&s_counts[my_sel], 1);
    }
    if (topk_score_out) {
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        const int e = j * 32 + lane;
        if (e < E) topk_score_out[(long long)t * E + e] = s[j];
      }
    }
  }
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

// aux = coeff * E * sum_i f_i P_i ;  aux_grad[i] = coeff * E * f_i / T  (dL/ds_ti)
__global__ void finalize_kernel(const int* __restrict__ counts,
                                const float* __restrict__ score_partials, int P, int T, int K,
                                int E, float coeff, float* __restrict__ aux_out,
                                float* __restrict__ aux_grad, float* __restrict__ mean_scores) {
  __shared__ double red[32];
  double local = 0.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    double ps = 0.0;
    for (int b = 0; b < P; ++b) ps += score_partials[(long long)b * E + e];
    const double Pm = ps / (double)(T > 0 ? T : 1);
    const double f = (double)counts[e] / (double)((long long)T * K > 0 ? (long long)T * K : 1);
    local += f * Pm;
    if (aux_grad) aux_grad[e] = (float)(coeff * E * f / (double)(T > 0 ? T : 1));
    if (mean_scores) mean_scores[e] = (float)Pm;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane_id() == 0) red[warp_id()] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) tot += red[w];
    *aux_out = (float)(coeff * E * tot);
  }
}

// dl = J_score^T ds with ds_te = dprob[t,k] (selected) + aux_grad[e]; written as bf16,
// zero-padded to ldd columns (the operand of the router wgrad / dgrad GEMMs).
template <int EPL>
__global__ void __launch_bounds__(WARPS * 32) bwd_kernel(
    const float* __restrict__ logits, int ld, int T, int E, int K, int score_fn,
    const int* __restrict__ topk_idx, const float* __restrict__ dprob,
    const float* __restrict__ aux_grad, __nv_bfloat16* __restrict__ dlogits, int ldd) {
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
    __nv_bfloat16* out = dlogits + (long long)t * ldd;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      float dl;
      if (score_fn == 0)
        dl = s[j] * (ds[j] - inner);
      else
        dl = sig[j] * (1.0f - sig[j]) * inv * (ds[j] - inner);
      if (e < E) out[e] = __float2bfloat16_rn(dl);
    }
    for (int e = E + lane; e < ldd; e += 32) out[e] = __float2bfloat16_rn(0.f);
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
  finalize_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      counts, score_partials, T == 0 ? 0 : P, T, K, E, coeff, aux_out, aux_grad, mean_scores);
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
  bwd_kernel<N><<<blocks, WARPS * 32, 0, st>>>(logits, ld, T, E, K, score_fn, topk_idx, dprob, \
                                              aux_grad, out, ldd)
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

}  // extern "C"
