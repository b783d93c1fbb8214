// Token permutation (dispatch index + gather) and unpermute/combine (gather-reduce),
// forward and backward. All data movement is 16-byte vectorised, one warp per token or
// row; all index construction is deterministic (ballot ranks + prefix sums, no
// atomics-ordered slots), so row maps are bit-exact against the oracle.
//
// Oracle: reference pkg/src/moelab/routing.py
//   permute          :149-168 (expert-major, ascending token, dropped skipped, phantom
//                              rows appended per expert, phantom rows zero)
//   unpermute_sum    :171-177 (per token, expert-ascending accumulation)
//   combine_standard :189-201 (prob multiplies the expert-output row, then sum)
//   combine_mem_eff. :204-223 (unweighted sum of rows that already carry p)
//   apply_capacity   :226-247 (keep first C selections per expert by token index; pad)
//   residual         :254-262 (+x for tokens whose every selection was dropped)
//
// Internal layout ("padded plan"): each expert's rows start at a multiple of 128
// (the grouped-GEMM M tile), rows [off_pad[e] + eff[e], off_pad[e+1]) are zero padding;
// phantom (capacity-pad) rows are the first padding rows of the block, exactly as in the
// oracle, so the oracle row_id_map is the concatenation of each block's first eff[e] rows.
#include "common.cuh"

namespace moe {
namespace perm {

constexpr int ALIGN = 128;

// P1: per-warp (32-token chunk) expert histograms + rank of each selection inside the chunk.
template <int KMAX>
__global__ void hist_kernel(const int* __restrict__ topk_idx, int T, int K, int E,
                            int* __restrict__ hist /*[W, E]*/, int* __restrict__ rank /*[T,K]*/) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int W = ceil_div_i(T, 32);
  if (gw >= W) return;
  const int t = gw * 32 + lane;
  const bool valid = t < T;
  const int* my = topk_idx + (long long)t * K;
  int sel[KMAX > 0 ? KMAX : 1];
  if constexpr (KMAX > 0) {
#pragma unroll
    for (int k = 0; k < KMAX; ++k) sel[k] = (valid && k < K) ? my[k] : -1;
  }
  const unsigned lt = (1u << lane) - 1u;
  for (int e = 0; e < E; ++e) {
    int which = -1;
    if constexpr (KMAX > 0) {
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (sel[k] == e) which = k;
    } else {
      if (valid)
        for (int k = 0; k < K; ++k)
          if (__ldg(my + k) == e) which = k;
    }
    const unsigned m = __ballot_sync(0xffffffffu, which >= 0);
    if (lane == 0) hist[(long long)gw * E + e] = __popc(m);
    if (which >= 0) rank[(long long)t * K + which] = __popc(m & lt);
  }
}

// P2: one warp per expert: exclusive scan over chunks -> base[w, e]; total count[e].
__global__ void scan_kernel(const int* __restrict__ hist, int W, int E, int* __restrict__ base,
                            int* __restrict__ count) {
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  if (e >= E) return;
  int run = 0;
  for (int w0 = 0; w0 < W; w0 += 32) {
    const int w = w0 + lane;
    const int v = w < W ? hist[(long long)w * E + e] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    if (w < W) base[(long long)w * E + e] = run + incl - v;
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) count[e] = run;
}

// P3: block offsets. capacity < 0 = dropless. meta layout (int32):
//   [0] num_m_blocks  [1] total padded rows  [2] total compact rows (sum eff)
//   off_pad[E+1], off_c[E+1], kept[E], eff[E]
__global__ void offsets_kernel(const int* __restrict__ count, int E, int capacity,
                               const int* __restrict__ cap_e, int pad,
                               const int* __restrict__ phantom, int align, int max_rows,
                               int* __restrict__ meta, int* __restrict__ off_pad,
                               int* __restrict__ off_c, int* __restrict__ kept,
                               int* __restrict__ eff, int* __restrict__ block_expert,
                               int* __restrict__ status) {
  __shared__ int s_pad[1025], s_c[1025];
  const int e = threadIdx.x;
  int kp = 0, ef = 0, pd = 0;
  if (e < E) {
    const int c = count[e];
    // per-expert capacity (EP global-position drops) or a uniform one
    const int cap = cap_e ? cap_e[e] : capacity;
    kp = cap < 0 ? c : min(c, cap);
    // phantom rows: explicit (routing_map_pad, routing.py:312-325) or capacity pad (:244-246)
    ef = phantom ? kp + phantom[e] : ((cap >= 0 && pad) ? cap : kp);
    pd = ceil_div_i(ef, align) * align;
    kept[e] = kp;
    eff[e] = ef;
  }
  s_pad[e] = pd;
  s_c[e] = ef;
  __syncthreads();
  // Hillis-Steele inclusive scan over blockDim.x entries (E <= 1024)
  for (int o = 1; o < blockDim.x; o <<= 1) {
    const int a = e >= o ? s_pad[e - o] : 0;
    const int b = e >= o ? s_c[e - o] : 0;
    __syncthreads();
    s_pad[e] += a;
    s_c[e] += b;
    __syncthreads();
  }
  if (e < E) {
    off_pad[e + 1] = s_pad[e];
    off_c[e + 1] = s_c[e];
  }
  if (e == 0) {
    off_pad[0] = 0;
    off_c[0] = 0;
    const int tot = s_pad[E - 1];
    if (tot > max_rows) atomicOr(status, 2);
    meta[0] = align >= ALIGN ? min(tot, max_rows) / ALIGN : 0;
    meta[1] = tot;
    meta[2] = s_c[E - 1];
  }
  __syncthreads();
  if (e < E && block_expert && align >= ALIGN) {
    const int b0 = (e ? s_pad[e - 1] : 0) / ALIGN;
    const int b1 = min(s_pad[e], max_rows) / ALIGN;
    for (int b = b0; b < b1; ++b) block_expert[b] = e;
  }
}

// P4: destination of every (token, k) selection + per-row source token and prob.
__global__ void assign_kernel(const int* __restrict__ topk_idx, const float* __restrict__ topk_prob,
                              const int* __restrict__ rank, const int* __restrict__ base, int T,
                              int K, int E, int capacity, const int* __restrict__ cap_e,
                              const int* __restrict__ off_pad, int max_rows,
                              int* __restrict__ inv_map, int* __restrict__ row_src,
                              float* __restrict__ row_prob) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)T * K) return;
  const int t = (int)(i / K);
  const int e = topk_idx[i];
  if (e < 0 || e >= E) {  // unused selection slot (ragged user-built routing maps)
    inv_map[i] = -1;
    return;
  }
  const int pos = base[(long long)(t >> 5) * E + e] + rank[i];
  int dest = -1;
  const int cap = cap_e ? cap_e[e] : capacity;
  if (cap < 0 || pos < cap) {
    dest = off_pad[e] + pos;
    if (dest < max_rows) {
      row_src[dest] = t;
      if (row_prob) row_prob[dest] = topk_prob ? topk_prob[i] : 1.0f;
    } else {
      dest = -1;
    }
  }
  inv_map[i] = dest;
}

// Padding / phantom rows of the plan: row_src = -1, row_prob = 0.
__global__ void pad_rows_kernel(const int* __restrict__ meta, const int* __restrict__ block_expert,
                                const int* __restrict__ off_pad, const int* __restrict__ kept,
                                int* __restrict__ row_src, float* __restrict__ row_prob) {
  const int rows = meta[0] * ALIGN;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const int e = block_expert[r / ALIGN];
    if (r - off_pad[e] >= kept[e]) {
      row_src[r] = -1;
      if (row_prob) row_prob[r] = 0.f;
    }
  }
}

// Split units of a 128-row aligned padded plan (the grouped GEMMs' kFlagSplit): expert e's
// blocks [off_pad[e] / 128, off_pad[e+1] / 128) become floor(n_e / 2) 256-row pairs and, when
// n_e is odd, one single 128-row block (its last). One block of 1024 threads; block order is
// preserved in both lists. U[0] = pairs, U[1] = singles, U[2 .. 2+cap) = pair start blocks,
// U[2+cap .. 2+2cap) = single blocks.
__global__ void split_units_kernel(const int* __restrict__ meta,
                                   const int* __restrict__ block_expert,
                                   const int* __restrict__ off_pad, int cap, int* __restrict__ U) {
  __shared__ int s_pair[1024], s_single[1024];
  const int nb = min(meta[0], cap);
  const int per = (cap + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  auto kind = [&](int b) {  // 1 = pair start, 2 = single, 0 = neither
    const int e = __ldg(block_expert + b);
    const int first = __ldg(off_pad + e) / ALIGN, end = __ldg(off_pad + e + 1) / ALIGN;
    if ((b - first) & 1) return 0;
    return b + 1 < end ? 1 : 2;
  };
  int np = 0, ns = 0;
  for (int b = b0; b < b1; ++b) {
    const int k = kind(b);
    np += k == 1;
    ns += k == 2;
  }
  s_pair[threadIdx.x] = np;
  s_single[threadIdx.x] = ns;
  __syncthreads();
  // exclusive scans (Hillis-Steele over 1024 entries)
  for (int off = 1; off < blockDim.x; off <<= 1) {
    const int a = threadIdx.x >= off ? s_pair[threadIdx.x - off] : 0;
    const int c = threadIdx.x >= off ? s_single[threadIdx.x - off] : 0;
    __syncthreads();
    s_pair[threadIdx.x] += a;
    s_single[threadIdx.x] += c;
    __syncthreads();
  }
  int ip = s_pair[threadIdx.x] - np, is = s_single[threadIdx.x] - ns;
  for (int b = b0; b < b1; ++b) {
    const int k = kind(b);
    if (k == 1) U[2 + ip++] = b;
    if (k == 2) U[2 + cap + is++] = b;
  }
  if (threadIdx.x == blockDim.x - 1) {
    U[0] = s_pair[threadIdx.x];
    U[1] = s_single[threadIdx.x];
  }
}

// compact (oracle-layout) map: compact row j of expert e = padded row off_pad[e] + (j - off_c[e])
__global__ void compact_map_kernel(const int* __restrict__ meta, const int* __restrict__ off_c,
                                   const int* __restrict__ off_pad, int E,
                                   const int* __restrict__ row_src, long long* __restrict__ out,
                                   int* __restrict__ compact_to_pad) {
  const int n = meta[2];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    int lo = 0, hi = E - 1;  // last e with off_c[e] <= j
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off_c[mid] <= j) lo = mid; else hi = mid - 1;
    }
    const int r = off_pad[lo] + (j - off_c[lo]);
    if (out) out[j] = row_src[r];
    if (compact_to_pad) compact_to_pad[j] = r;
  }
}

// Token-driven gather: read x[t] once, write it to each kept destination row.
template <int VPL>  // int4 vectors per lane per chunk
__global__ void gather_tokens_kernel(const int4* __restrict__ x, int T, int K, int hv /*int4/row*/,
                                     const int* __restrict__ inv_map, int4* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    const int* inv = inv_map + (long long)t * K;
    const int4* src = x + (long long)t * hv;
    for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
      int4 v[VPL];
      bool loaded = false;
      for (int k = 0; k < K; ++k) {
        const int d = __ldg(inv + k);
        if (d < 0) continue;
        if (!loaded) {
#pragma unroll
          for (int u = 0; u < VPL; ++u) {
            const int c = c0 + u * 32 + lane;
            if (c < hv) v[u] = ld_nc_v4(src + c);
          }
          loaded = true;
        }
        int4* o = out + (long long)d * hv;
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) st_na_v4(o + c, v[u]);
        }
      }
    }
  }
}

// Token-driven gather with the destination rows held in registers (K <= KMAX) and the next
// chunk of x loaded while the current one is stored K times (one load always in flight).
template <int VPL, int KMAX>
__global__ void gather_tokens_pf_kernel(const int4* __restrict__ x, int T, int K, int hv,
                                        const int* __restrict__ inv_map,
                                        int4* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  constexpr int CH = 32 * VPL;
  for (int t = warp; t < T; t += nwarps) {
    int d[KMAX];
    bool any = false;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      d[k] = k < K ? __ldg(inv_map + (long long)t * K + k) : -1;
      any |= d[k] >= 0;
    }
    if (!any) continue;
    const int4* src = x + (long long)t * hv;
    int4 cur[VPL], nxt[VPL];
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      const int c = u * 32 + lane;
      if (c < hv) cur[u] = ld_nc_v4(src + c);
    }
    for (int c0 = 0; c0 < hv; c0 += CH) {
      const bool more = c0 + CH < hv;
      if (more) {
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + CH + u * 32 + lane;
          if (c < hv) nxt[u] = ld_nc_v4(src + c);
        }
      }
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (d[k] < 0) continue;
        int4* o = out + (long long)d[k] * hv;
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) st_na_v4(o + c, cur[u]);
        }
      }
      if (more) {
#pragma unroll
        for (int u = 0; u < VPL; ++u) cur[u] = nxt[u];
      }
    }
  }
}

// Token-driven gather over (token, chunk) work items: a chunk is 32 lanes x VPL 16-byte
// vectors of one x row, read once and stored to each kept destination row. Splitting rows
// into chunks keeps every SM busy when T is small (DeepSeek shape: 4096 tokens of 14 KB).
template <int VPL>
__global__ void gather_chunks_kernel(const int4* __restrict__ x, int T, int K, int hv,
                                     const int* __restrict__ inv_map, int4* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int per_row = (hv + 32 * VPL - 1) / (32 * VPL);
  const long long items = (long long)T * per_row;
  for (long long it = warp; it < items; it += nwarps) {
    const int t = static_cast<int>(it / per_row);
    const int c0 = static_cast<int>(it - (long long)t * per_row) * 32 * VPL;
    const int* inv = inv_map + (long long)t * K;
    int4 v[VPL];
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      const int c = c0 + u * 32 + lane;
      if (c < hv) v[u] = ld_nc_v4(x + (long long)t * hv + c);
    }
    for (int k = 0; k < K; ++k) {
      const int d = __ldg(inv + k);
      if (d < 0) continue;
      int4* o = out + (long long)d * hv;
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < hv) st_na_v4(o + c, v[u]);
      }
    }
  }
}

// Token-driven gather on the TMA engine: each warp's lane 0 streams tokens, one bulk copy of
// the x row into shared memory (double-buffered, mbarrier completion) and one bulk store of
// it to each kept destination row. A write-dominated copy (K rows written per row read)
// issued as a handful of large asynchronous copies instead of K x hv 16-byte stores per
// token; the warp's other lanes idle.
constexpr int GT_WARPS = 4;
__global__ void __launch_bounds__(GT_WARPS * 32) gather_tokens_tma_kernel(
    const uint8_t* __restrict__ x, int T, int K, int row_bytes, const int* __restrict__ inv_map,
    uint8_t* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t gt_smem[];
  __shared__ __align__(8) uint64_t bars[GT_WARPS][2];
  const int warp = warp_id(), lane = lane_id();
  uint8_t* buf = gt_smem + warp * 2 * row_bytes;
  if (lane == 0) {
    mbar_init(&bars[warp][0], 1);
    mbar_init(&bars[warp][1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane != 0) return;
  const int nwarps = gridDim.x * GT_WARPS;
  // a token whose selections were all dropped has nothing to copy: skip its load
  auto next_token = [&](int t) {
    for (; t < T; t += nwarps) {
      for (int k = 0; k < K; ++k)
        if (__ldg(inv_map + (long long)t * K + k) >= 0) return t;
    }
    return t;
  };
  uint32_t ph = 0;
  int t = next_token(blockIdx.x * GT_WARPS + warp);
  if (t < T) {
    mbar_arrive_expect_tx(&bars[warp][0], row_bytes);
    bulk_load_g2s(buf, x + (long long)t * row_bytes, row_bytes, &bars[warp][0]);
  }
  for (int i = 0; t < T; ++i) {
    const int b = i & 1;
    const int tn = next_token(t + nwarps);
    // the other buffer's stores (token i-1) must have read it before it is refilled
    bulk_wait_read_0();
    if (tn < T) {
      mbar_arrive_expect_tx(&bars[warp][b ^ 1], row_bytes);
      bulk_load_g2s(buf + (b ^ 1) * row_bytes, x + (long long)tn * row_bytes, row_bytes,
                    &bars[warp][b ^ 1]);
    }
    mbar_wait(&bars[warp][b], (ph >> b) & 1);
    ph ^= 1u << b;
    for (int k = 0; k < K; ++k) {
      const int d = __ldg(inv_map + (long long)t * K + k);
      if (d >= 0) bulk_store_s2g(out + (long long)d * row_bytes, buf + b * row_bytes, row_bytes);
    }
    bulk_commit();
    t = tn;
  }
  bulk_wait_all();
}

// Zero the rows whose source is -1 (padding / phantom) among the first meta[0]*128 rows.
// Each warp checks 32 rows per step with 32 independent loads (lane l: row w + l * nwarps,
// so the padding rows, which sit together at the end of each expert block, spread over all
// warps), a ballot picks the padding rows, and the warp zeroes them: the scan is not a chain
// of one dependent 4-byte load per row (Qwen3 shape: ~270k rows).
__global__ void zero_pad_rows_kernel(const int* __restrict__ meta, const int* __restrict__ row_src,
                                     int hv, int4* __restrict__ out) {
  const int rows = meta[0] * ALIGN;
  const int lane = lane_id();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int4 z = make_int4(0, 0, 0, 0);
  for (long long base = warp; base < rows; base += 32LL * nwarps) {
    const long long r = base + (long long)lane * nwarps;
    unsigned m = __ballot_sync(0xffffffffu, r < rows && __ldg(row_src + r) < 0);
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      int4* o = out + (base + (long long)j * nwarps) * hv;
      for (int c = lane; c < hv; c += 32) st_na_v4(o + c, z);
    }
  }
}

// Dest-driven gather: out[r] = in[map[r]] (zero when map[r] < 0), r < n (n from device or host).
__global__ void gather_rows_kernel(const int4* __restrict__ in, int hv, const int* __restrict__ map,
                                   const int* __restrict__ n_dev, int n_host,
                                   int4* __restrict__ out) {
  const int n = n_dev ? *n_dev : n_host;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int4 z = make_int4(0, 0, 0, 0);
  for (int r = warp; r < n; r += nwarps) {
    const int s = __ldg(map + r);
    int4* o = out + (long long)r * hv;
    if (s < 0) {
      for (int c = lane_id(); c < hv; c += 32) st_na_v4(o + c, z);
    } else {
      const int4* i = in + (long long)s * hv;
      for (int c = lane_id(); c < hv; c += 32) st_na_v4(o + c, ld_nc_v4(i + c));
    }
  }
}

__device__ __forceinline__ void acc8(float (&a)[8], int4 v, float w, bool weighted) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = unpack_bf16x2(u[j]);
    // separate rounding of multiply and add: no FMA contraction (oracle order, routing.py:200)
    const float x0 = weighted ? __fmul_rn(f.x, w) : f.x;
    const float x1 = weighted ? __fmul_rn(f.y, w) : f.y;
    a[2 * j] = __fadd_rn(a[2 * j], x0);
    a[2 * j + 1] = __fadd_rn(a[2 * j + 1], x1);
  }
}
__device__ __forceinline__ int4 pack8(const float (&a)[8]) {
  int4 o;
  o.x = pack_bf16x2(a[0], a[1]);
  o.y = pack_bf16x2(a[2], a[3]);
  o.z = pack_bf16x2(a[4], a[5]);
  o.w = pack_bf16x2(a[6], a[7]);
  return o;
}

// Combine forward (gather-reduce): y[t] = sum_k w_k rows[inv[t,k]] (+ x[t] if all dropped),
// k in expert-ascending order; w_k = topk_prob (standard) or 1 (mem-efficient / unpermute).
// Also serves as the backward of permute (dX = unweighted sum of dXp rows) with `extra`
// (router dX contribution, added) and the residual taken from `resid` (dY).
template <int VPL>
__global__ void combine_kernel(const int4* __restrict__ rows, int T, int K, int hv,
                               const int* __restrict__ inv_map, const float* __restrict__ weights,
                               const int4* __restrict__ resid, const int4* __restrict__ extra,
                               const int4* __restrict__ extra2, int4* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    const int* inv = inv_map + (long long)t * K;
    bool any = false;
    for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
      float a[VPL][8];
#pragma unroll
      for (int u = 0; u < VPL; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[u][j] = 0.f;
      for (int k = 0; k < K; ++k) {
        const int d = __ldg(inv + k);
        if (d < 0) continue;
        any = true;
        const float w = weights ? __ldg(weights + (long long)t * K + k) : 1.0f;
        const int4* r = rows + (long long)d * hv;
        int4 v[VPL];
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) v[u] = ld_nc_v4(r + c);
        }
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) acc8(a[u], v[u], w, weights != nullptr);
        }
      }
      if (extra) {
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) acc8(a[u], ld_nc_v4(extra + (long long)t * hv + c), 1.f, false);
        }
      }
      if (extra2) {
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) acc8(a[u], ld_nc_v4(extra2 + (long long)t * hv + c), 1.f, false);
        }
      }
      if (!any && resid) {
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) acc8(a[u], ld_nc_v4(resid + (long long)t * hv + c), 1.f, false);
        }
      }
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < hv) st_na_v4(out + (long long)t * hv + c, pack8(a[u]));
      }
    }
  }
}

// Combine forward, K <= KMAX: the same sum as combine_kernel (same expert-ascending order,
// same separate multiply / add rounding, so bit-identical results), but every kept row's
// chunk is loaded before any is accumulated, so a warp has K row loads in flight instead of
// one dependent load per selection (top-8 at Qwen3 shape: 8x the memory-level parallelism).
template <int VPL, int KMAX>
__global__ void combine_mlp_kernel(const int4* __restrict__ rows, int T, int K, int hv,
                                   const int* __restrict__ inv_map,
                                   const float* __restrict__ weights,
                                   const int4* __restrict__ resid, const int4* __restrict__ extra,
                                   const int4* __restrict__ extra2, int4* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    int dst[KMAX];
    float w[KMAX];
    bool any = false;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      dst[k] = k < K ? __ldg(inv_map + (long long)t * K + k) : -1;
      w[k] = (weights && dst[k] >= 0) ? __ldg(weights + (long long)t * K + k) : 1.0f;
      any |= dst[k] >= 0;
    }
    for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
      int4 v[KMAX][VPL];
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (dst[k] >= 0 && c < hv) v[k][u] = ld_nc_v4(rows + (long long)dst[k] * hv + c);
        }
      int4 ex[VPL], ex2[VPL], rs[VPL];
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int c = c0 + u * 32 + lane;
        if (extra && c < hv) ex[u] = ld_nc_v4(extra + (long long)t * hv + c);
        if (extra2 && c < hv) ex2[u] = ld_nc_v4(extra2 + (long long)t * hv + c);
        if (!any && resid && c < hv) rs[u] = ld_nc_v4(resid + (long long)t * hv + c);
      }
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c >= hv) continue;
        float a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = 0.f;
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (dst[k] >= 0) acc8(a, v[k][u], w[k], weights != nullptr);
        if (extra) acc8(a, ex[u], 1.f, false);
        if (extra2) acc8(a, ex2[u], 1.f, false);
        if (!any && resid) acc8(a, rs[u], 1.f, false);
        st_na_v4(out + (long long)t * hv + c, pack8(a));
      }
    }
  }
}

// Combine backward, K <= KMAX (token-major): each dY chunk is read ONCE per token and the K
// expert-output rows of the chunk are loaded together; per selection
//   dO[dest] = p * dY[t]          (bf16, input of the fc2 dgrad / wgrad)
//   dprob[t,k] = <dY[t], O[dest]> (fp32; 0 for dropped selections)
// With O == NULL (mem-efficient combine) it only scatters dY unscaled.
template <int VPL, int KMAX>
__global__ void combine_bwd_mlp_kernel(const int4* __restrict__ dy,
                                       const int4* __restrict__ o_rows, int T, int K, int hv,
                                       const int* __restrict__ inv_map,
                                       const float* __restrict__ prob,
                                       int4* __restrict__ d_rows, float* __restrict__ dprob) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    int dst[KMAX];
    float p[KMAX], dot[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      dst[k] = k < K ? __ldg(inv_map + (long long)t * K + k) : -1;
      p[k] = (prob && dst[k] >= 0) ? __ldg(prob + (long long)t * K + k) : 1.f;
      dot[k] = 0.f;
    }
    for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
      int4 y[VPL], ov[KMAX][VPL];
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < hv) y[u] = ld_nc_v4(dy + (long long)t * hv + c);
      }
      if (o_rows) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
#pragma unroll
          for (int u = 0; u < VPL; ++u) {
            const int c = c0 + u * 32 + lane;
            if (dst[k] >= 0 && c < hv) ov[k][u] = ld_nc_v4(o_rows + (long long)dst[k] * hv + c);
          }
      }
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (dst[k] < 0) continue;
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c >= hv) continue;
          const uint32_t* uy = reinterpret_cast<const uint32_t*>(&y[u]);
          int4 wv;
          uint32_t* uw = reinterpret_cast<uint32_t*>(&wv);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 a = unpack_bf16x2(uy[j]);
            if (o_rows) {
              const float2 b = unpack_bf16x2(reinterpret_cast<const uint32_t*>(&ov[k][u])[j]);
              dot[k] += a.x * b.x + a.y * b.y;
            }
            uw[j] = prob ? pack_bf16x2(a.x * p[k], a.y * p[k]) : uy[j];
          }
          st_na_v4(d_rows + (long long)dst[k] * hv + c, wv);
        }
      }
    }
    if (dprob) {
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k >= K) break;
        const float s = warp_sum(dot[k]);
        if (lane == 0) dprob[(long long)t * K + k] = (dst[k] >= 0 && o_rows) ? s : 0.f;
      }
    }
  }
}

// Combine backward, any K (selection-major fallback).
__global__ void combine_bwd_kernel(const int4* __restrict__ dy, const int4* __restrict__ o_rows,
                                   int T, int K, int hv, const int* __restrict__ inv_map,
                                   const float* __restrict__ prob, int4* __restrict__ d_rows,
                                   float* __restrict__ dprob) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    for (int k = 0; k < K; ++k) {
      const long long i = (long long)t * K + k;
      const int d = __ldg(inv_map + i);
      if (d < 0) {
        if (lane == 0 && dprob) dprob[i] = 0.f;
        continue;
      }
      const float p = prob ? __ldg(prob + i) : 1.0f;
      float dot = 0.f;
      const int4* yr = dy + (long long)t * hv;
      const int4* orow = o_rows ? o_rows + (long long)d * hv : nullptr;
      int4* dr = d_rows + (long long)d * hv;
      for (int c = lane; c < hv; c += 32) {
        const int4 v = ld_nc_v4(yr + c);
        const uint32_t* u = reinterpret_cast<const uint32_t*>(&v);
        if (orow) {
          const int4 ov = ld_nc_v4(orow + c);
          const uint32_t* uo = reinterpret_cast<const uint32_t*>(&ov);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 a = unpack_bf16x2(u[j]);
            const float2 b = unpack_bf16x2(uo[j]);
            dot += a.x * b.x + a.y * b.y;
          }
        }
        int4 w;
        if (prob) {
          uint32_t* uw = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 a = unpack_bf16x2(u[j]);
            uw[j] = pack_bf16x2(a.x * p, a.y * p);
          }
        } else {
          w = v;
        }
        st_na_v4(dr + c, w);
      }
      if (dprob && orow) {
        dot = warp_sum(dot);
        if (lane == 0) dprob[i] = dot;
      }
    }
  }
}

// dprob for the mem-efficient combine: sum of the fc2-dgrad epilogue row partials.
__global__ void dprob_from_partials_kernel(const int* __restrict__ inv_map, long long n,
                                           const float* __restrict__ partial, int ldp,
                                           float* __restrict__ dprob) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = inv_map[i];
  float s = 0.f;
  if (d >= 0)
    for (int j = 0; j < ldp; ++j) s += partial[(long long)d * ldp + j];
  dprob[i] = s;
}

static int sms() { return device_sms(); }

static int warp_grid(long long items, int warps_per_block = 8) {
  const long long blocks = ceil_div_ll(items > 0 ? items : 1, warps_per_block);
  const long long cap = (long long)sms() * 8;  // 64 warps resident per SM
  return (int)(blocks < cap ? blocks : cap);
}

}  // namespace perm
}  // namespace moe

using namespace moe;
using namespace moe::perm;

extern "C" {

// workspace ints needed by moe_permute_plan: hist/base [W,E] x2 + rank [T,K]
long long moe_permute_workspace_ints(int T, int K, int E) {
  const long long W = ceil_div_i(T > 0 ? T : 1, 32);
  return 2 * W * E + (long long)T * K;
}

// Build the dispatch plan from top-k indices (device only, no host sync).
//   capacity: -1 dropless, else uniform per-expert capacity C; cap_e (nullable) overrides it
//             per expert (EP: C_global minus lower ranks' counts); pad != 0: drop-and-pad
//   phantom (nullable): explicit extra zero rows per expert (routing_map_pad)
//   align: 128 = padded plan for the grouped GEMM, 1 = compact (EP send buffer)
//   outputs: meta[3], off_pad[E+1], off_c[E+1], kept[E], eff[E], counts[E],
//            block_expert[max_rows/128] (nullable), inv_map[T,K], row_src[max_rows],
//            row_prob[max_rows] (nullable)
//   status bit 1: plan exceeded max_rows (rows beyond are dropped; caller must size buffers)
int moe_permute_plan(const int* topk_idx, const float* topk_prob, int T, int K, int E,
                     int capacity, const int* cap_e, int pad, const int* phantom, int align,
                     int max_rows, int* meta, int* off_pad, int* off_c, int* kept, int* eff,
                     int* counts, int* block_expert, int* inv_map, int* row_src,
                     float* row_prob, int* workspace, int* status, void* stream) {
  if (E < 1 || E > 1024 || K < 1 || K > 32) return kErrInvalidArg;
  if (align != 1 && align != ALIGN && align != 2 * ALIGN) return kErrInvalidArg;
  if (align >= ALIGN && max_rows % align) return kErrInvalidArg;
  auto st = static_cast<cudaStream_t>(stream);
  const int W = ceil_div_i(T > 0 ? T : 1, 32);
  int* hist = workspace;
  int* base = hist + (long long)W * E;
  int* rank = base + (long long)W * E;
  MOE_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(int), st));
  if (T > 0) {
    if (K <= 8)
      hist_kernel<8><<<ceil_div_i(W * 32, 256), 256, 0, st>>>(topk_idx, T, K, E, hist, rank);
    else
      hist_kernel<0><<<ceil_div_i(W * 32, 256), 256, 0, st>>>(topk_idx, T, K, E, hist, rank);
    MOE_LAUNCH_CHECK();
    scan_kernel<<<ceil_div_i(E * 32, 256), 256, 0, st>>>(hist, W, E, base, counts);
    MOE_LAUNCH_CHECK();
  } else {
    MOE_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(int) * E, st));
  }
  int threads = 32;
  while (threads < E) threads <<= 1;
  offsets_kernel<<<1, threads, 0, st>>>(counts, E, capacity, cap_e, pad, phantom, align,
                                        max_rows, meta, off_pad, off_c, kept, eff, block_expert,
                                        status);
  MOE_LAUNCH_CHECK();
  if (T > 0) {
    const long long n = (long long)T * K;
    assign_kernel<<<(int)ceil_div_ll(n, 256), 256, 0, st>>>(topk_idx, topk_prob, rank, base, T, K,
                                                           E, capacity, cap_e, off_pad, max_rows,
                                                           inv_map, row_src, row_prob);
    MOE_LAUNCH_CHECK();
  }
  if (align >= ALIGN && block_expert) {
    pad_rows_kernel<<<sms() * 4, 256, 0, st>>>(meta, block_expert, off_pad, kept, row_src,
                                                row_prob);
    MOE_LAUNCH_CHECK();
  }
  return kOk;
}

// ---------------------------------------------------------------------------- EP regroup
// Map between the all-to-all receive layout [src rank][local expert][rows] and the local
// padded plan [local expert][src rank rows | phantom | pad].  Host-built table (int32):
//   kept[n*el] (rows src s sends for local expert e), recv_off[n*el] (row offset of chunk
//   (s,e) in the receive buffer), off_pad[el+1], real[el] (= sum_s kept[s][e]).
// map_pad[r] = receive row feeding padded row r, or -1 (phantom / padding: zero row);
// map_recv[i] = padded row of receive row i.
__global__ void regroup_map_kernel(const int* __restrict__ tab, int n, int el, int rows_pad,
                                   int* __restrict__ map_pad, int* __restrict__ map_recv) {
  const int* kept = tab;
  const int* recv_off = tab + n * el;
  const int* off_pad = recv_off + n * el;
  const int* real = off_pad + el + 1;
  const int rows_plan = off_pad[el];  // rows_pad may be a static upper bound
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows_pad;
       r += gridDim.x * blockDim.x) {
    if (r >= rows_plan) {
      map_pad[r] = -1;
      continue;
    }
    int lo = 0, hi = el - 1;  // last e with off_pad[e] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off_pad[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int e = lo;
    const int j = r - off_pad[e];
    int src_row = -1;
    if (j < real[e]) {
      int acc = 0;
      for (int s = 0; s < n; ++s) {
        const int k = kept[s * el + e];
        if (j < acc + k) {
          src_row = recv_off[s * el + e] + (j - acc);
          break;
        }
        acc += k;
      }
    }
    map_pad[r] = src_row;
    if (src_row >= 0 && map_recv) map_recv[src_row] = r;
  }
}

int moe_ep_regroup_map(const int* table, int n, int el, int rows_pad, int* map_pad,
                       int* map_recv, void* stream) {
  if (n < 1 || el < 1) return kErrInvalidArg;
  if (rows_pad <= 0) return kOk;
  regroup_map_kernel<<<ceil_div_i(rows_pad, 256) < sms() * 8 ? ceil_div_i(rows_pad, 256)
                                                              : sms() * 8,
                       256, 0, static_cast<cudaStream_t>(stream)>>>(table, n, el, rows_pad,
                                                                    map_pad, map_recv);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Destination address of every padded row of the expert rank's plan in its SOURCE rank's
// compact buffer: row (local expert e, source s, q-th of s's rows for e) ->
// peers[s] + (dst_off[s * el + e] + q) * row_bytes; padding / phantom rows -> 0.
__global__ void row_dst_kernel(const int* __restrict__ tab, int n, int el, int rows_pad,
                               const int* __restrict__ dst_off,
                               const unsigned long long* __restrict__ peers,
                               long long row_bytes, unsigned long long* __restrict__ row_dst) {
  const int* kept = tab;
  const int* off_pad = tab + 2 * n * el;
  const int* real = off_pad + el + 1;
  const int rows_plan = off_pad[el];  // rows_pad may be a static upper bound
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows_pad;
       r += gridDim.x * blockDim.x) {
    if (r >= rows_plan) {
      row_dst[r] = 0ull;
      continue;
    }
    int lo = 0, hi = el - 1;  // last e with off_pad[e] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off_pad[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int e = lo;
    const int j = r - off_pad[e];
    unsigned long long dst = 0ull;
    if (j < real[e]) {
      int acc = 0;
      for (int s = 0; s < n; ++s) {
        const int k = kept[s * el + e];
        if (j < acc + k) {
          dst = peers[s] + static_cast<unsigned long long>(dst_off[s * el + e] + (j - acc)) *
                               static_cast<unsigned long long>(row_bytes);
          break;
        }
        acc += k;
      }
    }
    row_dst[r] = dst;
  }
}

int moe_ep_row_dst(const int* table, int n, int el, int rows_pad, const int* dst_off,
                   const unsigned long long* peers, long long row_bytes,
                   unsigned long long* row_dst, void* stream) {
  if (n < 1 || el < 1 || row_bytes <= 0 || (row_bytes & 15)) return kErrInvalidArg;
  if (rows_pad <= 0) return kOk;
  const int g = ceil_div_i(rows_pad, 256);
  row_dst_kernel<<<g < sms() * 8 ? g : sms() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      table, n, el, rows_pad, dst_off, peers, row_bytes, row_dst);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Oracle-layout (compact) row_id_map (int64, -1 phantom) and compact->padded row index.
// Unit table of a 128-row aligned padded plan for the grouped GEMMs' split mode (kFlagSplit):
// U [2 + 2 * cap] int32, cap = the plan's max_rows / 128.
int moe_split_units(const int* meta, const int* block_expert, const int* off_pad, int cap,
                    int* U, void* stream) {
  if (cap < 1) return kErrInvalidArg;
  split_units_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(meta, block_expert,
                                                                        off_pad, cap, U);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_permute_compact_map(const int* meta, const int* off_c, const int* off_pad, int E,
                            const int* row_src, long long* row_id_map, int* compact_to_pad,
                            int max_compact, void* stream) {
  compact_map_kernel<<<sms() * 4, 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(meta, off_c, off_pad, E, row_src,
                                                            row_id_map, compact_to_pad);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Gather tokens into the padded plan: xp[dest] = x[t]; padding rows zeroed.
int moe_permute_gather(const void* x, int T, int K, int h, const int* inv_map, const int* row_src,
                       const int* meta, void* xp, void* stream) {
  if (h % 8) return kErrInvalidArg;
  auto st = static_cast<cudaStream_t>(stream);
  const int hv = h / 8;
  // Default: one warp per token row (measured best, tools/hbm_probe.py: Mixtral 0.77, Qwen3
  // 0.84 of HBM). MOE_B200_GATHER=chunks: (token, chunk) work items (Qwen3 0.79);
  // =tma: bulk-copy variant (Mixtral 0.75, Qwen3 0.79). DeepSeek's 0.55 is the zero fill of
  // the padding rows (experts of ~128 rows padded to 128-row blocks), not counted here.
  // =pf: destination rows in registers, next chunk prefetched (standalone +1-7%, in-step
  // neutral; profiles/r02_gather_pf_ab.txt).
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("MOE_B200_GATHER");
    mode = !e ? 2 : (e[0] == 't' && e[1] == 'm') ? 1 : (e[0] == 'c') ? 0
                 : (e[0] == 'p' && e[1] == 'f') ? 3 : 2;
  }
  const int use_tma = mode == 1;
  const int row_bytes = h * 2;
  const int smem = GT_WARPS * 2 * row_bytes;
  if (T > 0 && use_tma && smem <= 200 * 1024) {
    MOE_CUDA_CHECK(
        ensure_dyn_smem(reinterpret_cast<const void*>(gather_tokens_tma_kernel), smem));
    const int blocks_per_sm = smem <= 100 * 1024 ? 2 : 1;
    const int want = ceil_div_i(T, GT_WARPS);
    const int grid = want < blocks_per_sm * sms() ? want : blocks_per_sm * sms();
    gather_tokens_tma_kernel<<<grid, GT_WARPS * 32, smem, st>>>(
        static_cast<const uint8_t*>(x), T, K, row_bytes, inv_map, static_cast<uint8_t*>(xp));
    MOE_LAUNCH_CHECK();
  } else if (T > 0 && mode == 3 && K <= 8) {
    gather_tokens_pf_kernel<4, 8><<<warp_grid(T), 256, 0, st>>>(
        static_cast<const int4*>(x), T, K, hv, inv_map, static_cast<int4*>(xp));
    MOE_LAUNCH_CHECK();
  } else if (T > 0 && (mode == 2 || mode == 3)) {
    gather_tokens_kernel<4><<<warp_grid(T), 256, 0, st>>>(static_cast<const int4*>(x), T, K, hv,
                                                          inv_map, static_cast<int4*>(xp));
    MOE_LAUNCH_CHECK();
  } else if (T > 0) {
    const long long items = (long long)T * ceil_div_i(hv, 32 * 2);
    gather_chunks_kernel<2><<<warp_grid(items), 256, 0, st>>>(
        static_cast<const int4*>(x), T, K, hv, inv_map, static_cast<int4*>(xp));
    MOE_LAUNCH_CHECK();
  }
  zero_pad_rows_kernel<<<sms() * 8, 256, 0, st>>>(meta, row_src, hv, static_cast<int4*>(xp));
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Zero padding rows only (e.g. the dO buffer before the combine backward fills real rows).
int moe_zero_pad_rows(const int* meta, const int* row_src, int h, void* rows, void* stream) {
  if (h % 8) return kErrInvalidArg;
  zero_pad_rows_kernel<<<sms() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      meta, row_src, h / 8, static_cast<int4*>(rows));
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Generic dest-driven row gather (bf16 rows of width h): out[r] = in[map[r]] or 0.
int moe_gather_rows(const void* in, int h, const int* map, const int* n_dev, int n_host,
                    void* out, void* stream) {
  if (h % 8) return kErrInvalidArg;
  const long long n_cap = n_dev ? (long long)sms() * 64 : n_host;
  gather_rows_kernel<<<warp_grid(n_cap), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(in), h / 8, map, n_dev, n_host, static_cast<int4*>(out));
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Combine / unpermute: y[t] = sum_k w[t,k] * rows[inv[t,k]] (+resid[t] if no kept selection)
// (+extra[t]). weights NULL = unweighted; resid / extra may be NULL.
int moe_combine(const void* rows, int T, int K, int h, const int* inv_map, const float* weights,
                const void* resid, const void* extra, const void* extra2, void* out,
                void* stream) {
  if (h % 8) return kErrInvalidArg;
  if (T == 0) return kOk;
  auto st = static_cast<cudaStream_t>(stream);
  const auto* r = static_cast<const int4*>(rows);
  const auto* rs = static_cast<const int4*>(resid);
  const auto* x1 = static_cast<const int4*>(extra);
  const auto* x2 = static_cast<const int4*>(extra2);
  auto* o = static_cast<int4*>(out);
  const int hv = h / 8;
  if (K <= 2)
    combine_mlp_kernel<4, 2><<<warp_grid(T), 256, 0, st>>>(r, T, K, hv, inv_map, weights, rs, x1,
                                                          x2, o);
  else if (K <= 4)
    combine_mlp_kernel<2, 4><<<warp_grid(T), 256, 0, st>>>(r, T, K, hv, inv_map, weights, rs, x1,
                                                          x2, o);
  else if (K <= 8)
    combine_mlp_kernel<2, 8><<<warp_grid(T), 256, 0, st>>>(r, T, K, hv, inv_map, weights, rs, x1,
                                                          x2, o);
  else
    combine_kernel<4><<<warp_grid(T), 256, 0, st>>>(r, T, K, hv, inv_map, weights, rs, x1, x2, o);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Combine backward: d_rows[dest] = prob * dY[t] (prob NULL: unscaled); dprob[t,k] = <dY, O>.
int moe_combine_bwd(const void* dy, const void* o_rows, int T, int K, int h, const int* inv_map,
                    const float* prob, void* d_rows, float* dprob, void* stream) {
  if (h % 8) return kErrInvalidArg;
  if (T == 0) return kOk;
  auto st = static_cast<cudaStream_t>(stream);
  const auto* y = static_cast<const int4*>(dy);
  const auto* o = static_cast<const int4*>(o_rows);
  auto* d = static_cast<int4*>(d_rows);
  const int hv = h / 8;
  if (K <= 2)
    combine_bwd_mlp_kernel<4, 2><<<warp_grid(T), 256, 0, st>>>(y, o, T, K, hv, inv_map, prob, d,
                                                              dprob);
  else if (K <= 4)
    combine_bwd_mlp_kernel<4, 4><<<warp_grid(T), 256, 0, st>>>(y, o, T, K, hv, inv_map, prob, d,
                                                              dprob);
  else if (K <= 8)
    combine_bwd_mlp_kernel<2, 8><<<warp_grid(T), 256, 0, st>>>(y, o, T, K, hv, inv_map, prob, d,
                                                              dprob);
  else
    combine_bwd_kernel<<<warp_grid(T), 256, 0, st>>>(y, o, T, K, hv, inv_map, prob, d, dprob);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_dprob_from_partials(const int* inv_map, long long n, const float* partial, int ldp,
                            float* dprob, void* stream) {
  if (n == 0) return kOk;
  dprob_from_partials_kernel<<<(int)ceil_div_ll(n, 256), 256, 0,
                               static_cast<cudaStream_t>(stream)>>>(inv_map, n, partial, ldp,
                                                                    dprob);
  MOE_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"
