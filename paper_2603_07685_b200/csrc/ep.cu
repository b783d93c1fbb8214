// Expert-parallel exchange fused into the permute / combine kernels over NVLink peer memory.
//
// The all-to-all of the reference's EP model (pkg/src/moelab/perf.py:62-70 counts its bytes;
// PAPER.md:204-211 describes the dispatcher) is not a separate collective here: every rank
// holds symmetric (peer-mapped) row buffers, and
//   * dispatch  = the permute gather, but each token row is stored straight into the
//                 destination rank's padded expert plan (NVLink P2P stores);
//   * combine   = the unpermute/combine gather-reduce, but expert-output rows are loaded
//                 straight from the expert rank's buffer (NVLink P2P loads, K rows in
//                 flight per lane); the pulled rows are also kept in a local compact copy;
//   * backward  = the combine backward computes dprob against that local copy and pushes
//                 p*dY to the expert rank in the same pass; the dX combine pulls dXp rows.
// Destination rows: row = base[e] + inv_c[t,k], where inv_c is the row of the selection in
// the source rank's compact expert-major plan (moe_permute_plan, align 1) and base[e] is the
// host-computed offset of this source's block inside expert e's padded block on its rank
// (padded offset + rows of lower source ranks - compact offset), so the rows of expert e
// on its home rank are ordered (source rank, token) = global token order, exactly the
// oracle's permute order on the global batch (routing.py:155-163).
//
// Push kernels end with __threadfence_system(); cross-rank completion is established by a
// stream-ordered NCCL collective between the push and the consumer (no spin-waits).
// A negative destination row (base[e] + inv_c < 0) is skipped by every push and pull: the
// device planner poisons base[] that way when the EP group is inconsistent (token counts
// differ across ranks, or a plan exceeds the static buffers), so no rank ever stores past
// a peer's allocation; the status word it sets makes check_ep_status() raise.
#include "common.cuh"

namespace moe {
namespace ep {

__device__ __forceinline__ int4 ld_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void acc8(float (&a)[8], int4 v, float w, bool weighted) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = unpack_bf16x2(u[j]);
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

// Dispatch: x[t] -> peers[rank(e)][base[e] + inv_c[t,k]] for every kept selection.
template <int VPL>
__global__ void dispatch_push_kernel(const int4* __restrict__ x, int T, int K, int hv,
                                     const int* __restrict__ topk_idx,
                                     const int* __restrict__ inv_c,
                                     const int* __restrict__ base, int el,
                                     const unsigned long long* __restrict__ peers,
                                     const float* __restrict__ prob,
                                     const unsigned long long* __restrict__ prob_peers,
                                     int dest) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    const int4* src = x + (long long)t * hv;
    for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
      int4 v[VPL];
      bool loaded = false;
      for (int k = 0; k < K; ++k) {
        const int d = __ldg(inv_c + (long long)t * K + k);
        if (d < 0) continue;
        const int e = __ldg(topk_idx + (long long)t * K + k);
        const int r = e / el;
        if (dest >= 0 && r != dest) continue;
        const long long row = (long long)__ldg(base + e) + d;
        if (row < 0) continue;  // poisoned plan (moe_ep_plan_device: inconsistent EP group)
        if (!loaded) {
#pragma unroll
          for (int u = 0; u < VPL; ++u) {
            const int c = c0 + u * 32 + lane;
            if (c < hv) v[u] = ld_nc_v4(src + c);
          }
          loaded = true;
        }
        int4* dst = reinterpret_cast<int4*>(peers[r]) + row * hv;
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) dst[c] = v[u];
        }
        if (c0 == 0 && lane == 0 && prob_peers)
          reinterpret_cast<float*>(prob_peers[r])[row] = prob[(long long)t * K + k];
      }
    }
  }
  __threadfence_system();
}

// Combine (pull): y[t] = sum_k w_k * peers[rank(e)][base[e] + inv_c]  (+resid if no kept)
// (+extra, extra2); with rows_copy, each pulled row is also stored at rows_copy[inv_c].
// K <= KMAX: the K rows of a chunk are all loaded before any is accumulated (MLP).
template <int VPL, int KMAX>
__global__ void combine_pull_kernel(const unsigned long long* __restrict__ peers, int T, int K,
                                    int hv, const int* __restrict__ topk_idx,
                                    const int* __restrict__ inv_c,
                                    const int* __restrict__ base, int el,
                                    const float* __restrict__ weights,
                                    const int4* __restrict__ resid,
                                    const int4* __restrict__ extra,
                                    const int4* __restrict__ extra2, int4* __restrict__ out,
                                    int4* __restrict__ rows_copy) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    const int4* rows[KMAX];
    int4* copy[KMAX];
    float w[KMAX];
    bool any = false;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      rows[k] = nullptr;
      copy[k] = nullptr;
      w[k] = 0.f;
      if (k < K) {
        const int d = __ldg(inv_c + (long long)t * K + k);
        const int e = d >= 0 ? __ldg(topk_idx + (long long)t * K + k) : 0;
        if (d >= 0 && __ldg(base + e) + d >= 0) {  // (a poisoned plan pulls nothing)
          rows[k] = reinterpret_cast<const int4*>(peers[e / el]) +
                    ((long long)__ldg(base + e) + d) * hv;
          if (rows_copy) copy[k] = rows_copy + (long long)d * hv;
          w[k] = weights ? __ldg(weights + (long long)t * K + k) : 1.0f;
          any = true;
        }
      }
    }
    for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
      int4 v[KMAX][VPL];
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (rows[k] && c < hv) v[k][u] = ld_v4(rows[k] + c);
        }
      float a[VPL][8];
#pragma unroll
      for (int u = 0; u < VPL; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[u][j] = 0.f;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (rows[k] && c < hv) {
            acc8(a[u], v[k][u], w[k], weights != nullptr);
            if (copy[k]) st_na_v4(copy[k] + c, v[k][u]);
          }
        }
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c >= hv) continue;
        if (extra) acc8(a[u], ld_nc_v4(extra + (long long)t * hv + c), 1.f, false);
        if (extra2) acc8(a[u], ld_nc_v4(extra2 + (long long)t * hv + c), 1.f, false);
        if (!any && resid) acc8(a[u], ld_nc_v4(resid + (long long)t * hv + c), 1.f, false);
        st_na_v4(out + (long long)t * hv + c, pack8(a[u]));
      }
    }
  }
}

// Combine backward (push): per kept selection, p * dY[t] is stored into the expert rank's
// row and dprob = <dY[t], O row> is computed against the LOCAL compact copy of the expert
// output (o_local[inv_c], written by the forward pull). o_local NULL: mem-efficient
// combine (unscaled dY pushed, dprob comes from the expert rank's partials).
template <int VPL, int KMAX>
__global__ void combine_bwd_push_kernel(const int4* __restrict__ dy,
                                        const int4* __restrict__ o_local,
                                        const unsigned long long* __restrict__ d_peers, int T,
                                        int K, int hv, const int* __restrict__ topk_idx,
                                        const int* __restrict__ inv_c,
                                        const int* __restrict__ base, int el,
                                        const float* __restrict__ prob,
                                        float* __restrict__ dprob, int dest) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    const int4* orow[KMAX];
    int4* drow[KMAX];
    float p[KMAX], dot[KMAX];
    bool any = false;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      orow[k] = nullptr;
      drow[k] = nullptr;
      p[k] = 1.f;
      dot[k] = 0.f;
      if (k < K) {
        const long long i = (long long)t * K + k;
        const int d = __ldg(inv_c + i);
        const int e = d >= 0 ? __ldg(topk_idx + i) : -1;
        if (d >= 0 && (dest < 0 || e / el == dest) && __ldg(base + e) + d >= 0) {
          any = true;
          const long long row = (long long)__ldg(base + e) + d;
          if (o_local) orow[k] = o_local + (long long)d * hv;
          drow[k] = reinterpret_cast<int4*>(d_peers[e / el]) + row * hv;
          if (prob) p[k] = __ldg(prob + i);
        }
      }
    }
    if (dest >= 0 && !any) continue;  // no selection of this token goes to `dest`
    for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
      int4 y[VPL], ov[KMAX][VPL];
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < hv) y[u] = ld_nc_v4(dy + (long long)t * hv + c);
      }
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (orow[k] && c < hv) ov[k][u] = ld_nc_v4(orow[k] + c);
        }
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (!drow[k]) continue;
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
            if (orow[k]) {
              const float2 b = unpack_bf16x2(reinterpret_cast<const uint32_t*>(&ov[k][u])[j]);
              dot[k] += a.x * b.x + a.y * b.y;
            }
            uw[j] = prob ? pack_bf16x2(a.x * p[k], a.y * p[k]) : uy[j];
          }
          drow[k][c] = wv;
        }
      }
    }
    if (dprob) {
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k >= K) break;
        const float s = warp_sum(dot[k]);
        // per-destination passes write only their own selections (caller zero-fills)
        if (lane == 0 && (dest < 0 || drow[k]))
          dprob[(long long)t * K + k] = (drow[k] && o_local) ? s : 0.f;
      }
    }
  }
  __threadfence_system();
}

// Per-destination combine backward for the overlapped dispatch: the same math as
// combine_bwd_push_kernel, one selection at a time (dY re-read from L2 per selection), so it
// needs few registers. It runs beside a persistent GEMM whose 6 warps take up to 184
// registers each: warps are spread round-robin over the 4 SM sub-partitions (16K registers
// each), which leaves about 4.6K registers per sub-partition, i.e. <= 144 per thread here.
template <int VPL>
__global__ void __launch_bounds__(128) combine_bwd_push_sel_kernel(
    const int4* __restrict__ dy, const int4* __restrict__ o_local,
    const unsigned long long* __restrict__ d_peers, int T, int K, int hv,
    const int* __restrict__ topk_idx, const int* __restrict__ inv_c,
    const int* __restrict__ base, int el, const float* __restrict__ prob,
    float* __restrict__ dprob, int dest) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    for (int k = 0; k < K; ++k) {
      const long long i = (long long)t * K + k;
      const int d = __ldg(inv_c + i);
      if (d < 0) continue;
      const int e = __ldg(topk_idx + i);
      if (e / el != dest) continue;
      const long long row = (long long)__ldg(base + e) + d;
      if (row < 0) continue;
      int4* drow = reinterpret_cast<int4*>(d_peers[dest]) + row * hv;
      const int4* orow = o_local ? o_local + (long long)d * hv : nullptr;
      const float p = prob ? __ldg(prob + i) : 1.f;
      float dot = 0.f;
      for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
        int4 y[VPL], ov[VPL];
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) {
            y[u] = __ldg(dy + (long long)t * hv + c);
            if (orow) ov[u] = ld_nc_v4(orow + c);
          }
        }
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
            if (orow) {
              const float2 b = unpack_bf16x2(reinterpret_cast<const uint32_t*>(&ov[u])[j]);
              dot += a.x * b.x + a.y * b.y;
            }
            uw[j] = prob ? pack_bf16x2(a.x * p, a.y * p) : uy[j];
          }
          drow[c] = wv;
        }
      }
      if (dprob) {
        const float s = warp_sum(dot);
        if (lane == 0) dprob[i] = o_local ? s : 0.f;
      }
    }
  }
  __threadfence_system();
}

// dprob (mem-efficient combine): sum of the expert rank's fc2-dgrad row partials, pulled.
__global__ void dprob_pull_kernel(const unsigned long long* __restrict__ part_peers, long long n,
                                  int K, const int* __restrict__ topk_idx,
                                  const int* __restrict__ inv_c, const int* __restrict__ base,
                                  int el, int ldp, float* __restrict__ dprob) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = inv_c[i];
  float s = 0.f;
  const int e = d >= 0 ? topk_idx[i] : 0;
  if (d >= 0 && (long long)base[e] + d >= 0) {
    const long long row = (long long)base[e] + d;
    const float* pr = reinterpret_cast<const float*>(part_peers[e / el]) + row * ldp;
    for (int j = 0; j < ldp; ++j) s += pr[j];
  }
  dprob[i] = s;
}

// ---------------------------------------------------------------- token de-duplication
// (HybridEP-style; byte model perf.py:81-160): a token is sent ONCE to
// every destination rank that hosts at least one of its kept experts; the destination
// expands it to its expert rows locally and pre-reduces the token's expert outputs before
// the source pulls one row per (token, rank).

// Per token: distinct destination ranks of its kept selections (ascending, -1 padded), and
// per selection the index of its rank in that list and its position among the token's
// selections on that rank. Selections are ascending by expert, so ranks are non-decreasing.
__global__ void token_ranks_kernel(const int* __restrict__ topk_idx,
                                   const int* __restrict__ inv_c, int T, int K, int el,
                                   int* __restrict__ rank_idx, int* __restrict__ sel_j,
                                   int* __restrict__ sel_pos) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  int j = -1, pos = 0, last = -1;
  for (int k = 0; k < K; ++k) {
    const long long i = (long long)t * K + k;
    if (inv_c[i] < 0) {
      sel_j[i] = -1;
      sel_pos[i] = -1;
      continue;
    }
    const int r = topk_idx[i] / el;
    if (r != last) {
      ++j;
      pos = 0;
      last = r;
      rank_idx[(long long)t * K + j] = r;
    } else {
      ++pos;
    }
    sel_j[i] = j;
    sel_pos[i] = pos;
  }
  for (int jj = j + 1; jj < K; ++jj) rank_idx[(long long)t * K + jj] = -1;
}

// Dedup dispatch: x[t] -> tok_peers[d][tbase[d] + inv_rank[t,j]] once per distinct rank d,
// plus, per kept selection on d: expand map (expert row -> token row), the token row's
// slot table (row, prob) used by the destination's partial combine, and the row's prob.
template <int VPL>
__global__ void dispatch_dedup_kernel(const int4* __restrict__ x, int T, int K, int hv,
                                      const int* __restrict__ topk_idx,
                                      const int* __restrict__ inv_c,
                                      const int* __restrict__ base, int el,
                                      const int* __restrict__ rank_idx,
                                      const int* __restrict__ inv_rank,
                                      const int* __restrict__ tbase,
                                      const int* __restrict__ sel_j,
                                      const int* __restrict__ sel_pos,
                                      const float* __restrict__ prob,
                                      const unsigned long long* __restrict__ tok_peers,
                                      const unsigned long long* __restrict__ map_peers,
                                      const unsigned long long* __restrict__ srows_peers,
                                      const unsigned long long* __restrict__ sprob_peers,
                                      const unsigned long long* __restrict__ rprob_peers) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    const long long tk = (long long)t * K;
    // metadata: lane k handles selection k, lane j handles the -1 fill of rank slot j
    for (int k = lane; k < K; k += 32) {
      const int j = __ldg(sel_j + tk + k);
      if (j < 0) continue;
      const int e = __ldg(topk_idx + tk + k);
      const int d = e / el;
      const long long r = (long long)__ldg(base + e) + __ldg(inv_c + tk + k);
      const long long trow = (long long)__ldg(tbase + d) + __ldg(inv_rank + tk + j);
      const float p = prob ? __ldg(prob + tk + k) : 1.0f;
      reinterpret_cast<int*>(map_peers[d])[r] = (int)trow;
      reinterpret_cast<int*>(srows_peers[d])[trow * K + __ldg(sel_pos + tk + k)] = (int)r;
      reinterpret_cast<float*>(sprob_peers[d])[trow * K + __ldg(sel_pos + tk + k)] = p;
      reinterpret_cast<float*>(rprob_peers[d])[r] = p;
    }
    for (int j = lane; j < K; j += 32) {
      const int d = __ldg(rank_idx + tk + j);
      if (d < 0) continue;
      int cnt = 0;
      for (int k = 0; k < K; ++k) cnt += (__ldg(sel_j + tk + k) == j);
      const long long trow = (long long)__ldg(tbase + d) + __ldg(inv_rank + tk + j);
      for (int pos = cnt; pos < K; ++pos)
        reinterpret_cast<int*>(srows_peers[d])[trow * K + pos] = -1;
    }
    // the row itself, once per destination rank
    const int4* src = x + (long long)t * hv;
    for (int c0 = 0; c0 < hv; c0 += 32 * VPL) {
      int4 v[VPL];
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < hv) v[u] = ld_nc_v4(src + c);
      }
      for (int j = 0; j < K; ++j) {
        const int d = __ldg(rank_idx + tk + j);
        if (d < 0) break;
        const long long trow = (long long)__ldg(tbase + d) + __ldg(inv_rank + tk + j);
        int4* dst = reinterpret_cast<int4*>(tok_peers[d]) + trow * hv;
#pragma unroll
        for (int u = 0; u < VPL; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < hv) dst[c] = v[u];
        }
      }
    }
  }
  __threadfence_system();
}

// map[r] = -1 for the padding / phantom rows of the local plan (map_pad < 0); real rows
// are written by the sources' dedup dispatch (disjoint entries, no race).
__global__ void fill_pad_map_kernel(const int* __restrict__ map_pad, int rows,
                                    int* __restrict__ map) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    if (map_pad[r] < 0) map[r] = -1;
}

// Expert-side backward expansion: d_o[r] = p_r * tok[map[r]] (p_r = 1 without rowprob),
// dprob_rows[r] = <tok[map[r]], o[r]> (standard combine); zero rows where map[r] < 0.
__global__ void expand_grad_kernel(const int4* __restrict__ tok, const int* __restrict__ map,
                                   int rows, int hv, const float* __restrict__ rowprob,
                                   const int4* __restrict__ o, int4* __restrict__ d_o,
                                   float* __restrict__ dprob_rows) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int4 z = make_int4(0, 0, 0, 0);
  for (int r = warp; r < rows; r += nwarps) {
    const int s = __ldg(map + r);
    int4* dr = d_o + (long long)r * hv;
    if (s < 0) {
      for (int c = lane; c < hv; c += 32) st_na_v4(dr + c, z);
      if (lane == 0 && dprob_rows) dprob_rows[r] = 0.f;
      continue;
    }
    const float p = rowprob ? __ldg(rowprob + r) : 1.0f;
    const int4* tr = tok + (long long)s * hv;
    const int4* orow = o ? o + (long long)r * hv : nullptr;
    float dot = 0.f;
    for (int c = lane; c < hv; c += 32) {
      const int4 v = ld_nc_v4(tr + c);
      const uint32_t* u = reinterpret_cast<const uint32_t*>(&v);
      int4 w;
      uint32_t* uw = reinterpret_cast<uint32_t*>(&w);
      int4 ov;
      if (orow) ov = ld_nc_v4(orow + c);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = unpack_bf16x2(u[j]);
        if (orow) {
          const float2 b = unpack_bf16x2(reinterpret_cast<const uint32_t*>(&ov)[j]);
          dot += a.x * b.x + a.y * b.y;
        }
        uw[j] = rowprob ? pack_bf16x2(a.x * p, a.y * p) : u[j];
      }
      st_na_v4(dr + c, w);
    }
    if (dprob_rows) {
      dot = warp_sum(dot);
      if (lane == 0) dprob_rows[r] = orow ? dot : 0.f;
    }
  }
}

// ECHO (hot-expert cloning, reference planners.py:243-389): selection (t,k) of expert e at
// global position p = gbase[e] + inv_c[t,k] is served by the segment j with
// seg_start[e,j] <= p < seg_start[e,j+1]; its virtual expert is seg_v[e,j].
__global__ void echo_rewrite_kernel(const int* __restrict__ topk_idx,
                                    const int* __restrict__ inv_c, long long n, int ns,
                                    const int* __restrict__ gbase,
                                    const int* __restrict__ seg_start,
                                    const int* __restrict__ seg_v, int* __restrict__ topk_v) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = inv_c[i];
  if (d < 0) {
    topk_v[i] = -1;
    return;
  }
  const int e = topk_idx[i];
  const int p = gbase[e] + d;
  int v = seg_v[e * ns];
  for (int j = 1; j < ns; ++j) {
    const int s = seg_start[e * ns + j];
    if (s <= p && seg_v[e * ns + j] >= 0) v = seg_v[e * ns + j];
  }
  topk_v[i] = v;
}

static int sms() { return device_sms(); }
// Kernels that must run beside a persistent grouped GEMM (the overlapped dispatch) use the
// GEMM's L1/shared split: an SM only hosts CTAs of kernels whose carve-out matches its
// current configuration, so with the default (L1-preferring) carve-out a push CTA would wait
// for the GEMM to drain, and the GEMM waits for the push.
template <typename K>
static void prefer_max_shared(K kern) {
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                       static_cast<int>(cudaSharedmemCarveoutMaxShared));
}
static int warp_grid(long long items) {
  const long long blocks = ceil_div_ll(items > 0 ? items : 1, 8);
  const long long cap = (long long)sms() * 8;
  return (int)(blocks < cap ? blocks : cap);
}

}  // namespace ep
}  // namespace moe

using namespace moe;
using namespace moe::ep;

extern "C" {

int moe_ep_dispatch_push(const void* x, int T, int K, int h, const int* topk_idx,
                         const int* inv_c, const int* base, int el,
                         const unsigned long long* peers, const float* prob,
                         const unsigned long long* prob_peers, void* stream) {
  if (h % 8 || el < 1) return kErrInvalidArg;
  if (T == 0) return kOk;
  dispatch_push_kernel<4><<<warp_grid(T), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(x), T, K, h / 8, topk_idx, inv_c, base, el, peers, prob,
      prob_peers, -1);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Dispatch restricted to the selections whose expert lives on rank `dest`.
int moe_ep_dispatch_push_dest(const void* x, int T, int K, int h, const int* topk_idx,
                              const int* inv_c, const int* base, int el,
                              const unsigned long long* peers, const float* prob,
                              const unsigned long long* prob_peers, int dest, void* stream) {
  if (h % 8 || el < 1 || dest < 0) return kErrInvalidArg;
  if (T == 0) return kOk;
  dispatch_push_kernel<4><<<warp_grid(T), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(x), T, K, h / 8, topk_idx, inv_c, base, el, peers, prob,
      prob_peers, dest);
  MOE_LAUNCH_CHECK();
  return kOk;
}

__global__ void signal_kernel(const unsigned long long* __restrict__ flag_peers, int dest,
                              int slot, const uint32_t* __restrict__ epoch) {
  __threadfence_system();
  st_release_sys_u32(reinterpret_cast<uint32_t*>(flag_peers[dest]) + slot,
                     *reinterpret_cast<const volatile uint32_t*>(epoch));
}

__global__ void epoch_bump_kernel(uint32_t* epoch) { *epoch += 1u; }

// Publish "this rank's rows for `dest` are complete": flag_peers[dest][slot] = *epoch
// (release, system scope), ordered after the preceding pushes on `stream`.
int moe_ep_signal(const unsigned long long* flag_peers, int dest, int slot,
                  const unsigned int* epoch, void* stream) {
  if (dest < 0 || slot < 0 || !epoch) return kErrInvalidArg;
  signal_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag_peers, dest, slot, epoch);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Advance the dispatch epoch (device scalar) in stream order.
int moe_ep_epoch_bump(unsigned int* epoch, void* stream) {
  if (!epoch) return kErrInvalidArg;
  epoch_bump_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(epoch);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// rows[r] -> *row_dst[r] (0 = skip) for r < rows: the EP return transfer as a standalone
// NVLink push (warp per row, 512 contiguous bytes per instruction) for GEMMs without a
// scatter epilogue (the MXFP8 engine).
__global__ void scatter_rows_kernel(const int4* __restrict__ src, int rows, int hv,
                                    const unsigned long long* __restrict__ row_dst) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < rows; r += nwarps) {
    const unsigned long long d = __ldg(row_dst + r);
    if (!d) continue;
    int4* dst = reinterpret_cast<int4*>(d);
    const int4* s = src + (long long)r * hv;
    for (int c = lane; c < hv; c += 32) dst[c] = ld_nc_v4(s + c);
  }
  __threadfence_system();
}

int moe_ep_scatter_rows(const void* src, int rows, int h, const unsigned long long* row_dst,
                        void* stream) {
  if (h % 8 || rows < 0) return kErrInvalidArg;
  if (rows == 0) return kOk;
  scatter_rows_kernel<<<warp_grid(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(src), rows, h / 8, row_dst);
  MOE_LAUNCH_CHECK();
  return kOk;
}

// Per 128-row block of this rank's padded plan: bitmask of the source ranks whose rows it
// holds (table of moe_ep_regroup_map), and the schedule of GEMM units (unit = `cg` blocks)
// sorted by the arrival position of their latest source: source s pushes to ranks
// s, s+1, ... in turn, so rank `me` receives from me, me-1, me-2, ... in that order.
__global__ void block_need_kernel(const int* __restrict__ tab, int n, int el, int me,
                                  int nblocks, int cg, uint32_t* __restrict__ need,
                                  int* __restrict__ order) {
  const int* kept = tab;
  const int* off_pad = tab + 2 * n * el;
  const int* real = off_pad + el + 1;
  __shared__ int cnt[33];
  __shared__ int base_s[33];
  nblocks = min(nblocks, off_pad[el] / 128);  // nblocks may be a static upper bound
  const int nunits = nblocks / cg;
  if (threadIdx.x <= 32) cnt[threadIdx.x] = 0;
  __syncthreads();
  // pass 1: masks and per-priority unit counts
  for (int u = threadIdx.x; u < nunits; u += blockDim.x) {
    int pri = 0;
    for (int b = u * cg; b < (u + 1) * cg; ++b) {
      const int r0 = b * 128, r1 = r0 + 128;
      uint32_t m = 0;
      for (int e = 0; e < el; ++e) {
        const int lo = off_pad[e], hi = off_pad[e] + real[e];
        if (hi <= r0 || lo >= r1) continue;
        int acc = lo;
        for (int s = 0; s < n; ++s) {
          const int k = kept[s * el + e];
          if (k > 0 && acc < r1 && acc + k > r0) {
            m |= 1u << s;
            const int pr = (me - s + n) % n;
            pri = pr > pri ? pr : pri;
          }
          acc += k;
        }
      }
      need[b] = m;
    }
    atomicAdd(&cnt[pri], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int i = 0; i < n; ++i) {
      base_s[i] = a;
      a += cnt[i];
    }
  }
  __syncthreads();
  // pass 2: stable placement by priority (one warp per priority level keeps unit order)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int pl = w; pl < n; pl += blockDim.x >> 5) {
    int pos = base_s[pl];
    for (int u0 = 0; u0 < nunits; u0 += 32) {
      const int u = u0 + lane;
      bool hit = false;
      if (u < nunits) {
        int pri = 0;
        for (int b = u * cg; b < (u + 1) * cg; ++b) {
          const uint32_t m = need[b];
          for (int s = 0; s < n; ++s)
            if (m >> s & 1u) {
              const int pr = (me - s + n) % n;
              pri = pr > pri ? pr : pri;
            }
        }
        hit = pri == pl;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit) order[pos + __popc(bal & ((1u << lane) - 1u))] = u;
      pos += __popc(bal);
    }
  }
}

// Load and configure every kernel the overlapped dispatch launches beside a running GEMM.
// Must be called before the first overlapped step: with CUDA lazy loading, the first launch
// of a kernel may wait for the device's running kernels, i.e. for a GEMM that waits for it.
int moe_ep_prepare() {
  prefer_max_shared(dispatch_push_kernel<4>);
  prefer_max_shared(combine_bwd_push_sel_kernel<2>);
  prefer_max_shared(signal_kernel);
  prefer_max_shared(epoch_bump_kernel);
  cudaFuncAttributes a;
  MOE_CUDA_CHECK(cudaFuncGetAttributes(&a, epoch_bump_kernel));
  MOE_CUDA_CHECK(cudaFuncGetAttributes(&a, dispatch_push_kernel<4>));
  MOE_CUDA_CHECK(cudaFuncGetAttributes(&a, combine_bwd_push_sel_kernel<2>));
  MOE_CUDA_CHECK(cudaFuncGetAttributes(&a, signal_kernel));
  return kOk;
}

int moe_ep_block_need(const int* table, int n, int el, int me, int nblocks, int cg,
                      unsigned int* need, int* order, void* stream) {
  if (n < 1 || n > 32 || el < 1 || (cg != 1 && cg != 2) || nblocks % cg) return kErrInvalidArg;
  if (nblocks <= 0) return kOk;
  block_need_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(table, n, el, me, nblocks,
                                                                      cg, need, order);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_ep_combine_pull(const unsigned long long* peers, int T, int K, int h,
                        const int* topk_idx, const int* inv_c, const int* base, int el,
                        const float* weights, const void* resid, const void* extra,
                        const void* extra2, void* out, void* rows_copy, void* stream) {
  if (h % 8 || el < 1 || K > 32) return kErrInvalidArg;
  if (T == 0) return kOk;
  auto st = static_cast<cudaStream_t>(stream);
  const auto* r = static_cast<const int4*>(resid);
  const auto* x1 = static_cast<const int4*>(extra);
  const auto* x2 = static_cast<const int4*>(extra2);
  auto* o = static_cast<int4*>(out);
  auto* cp = static_cast<int4*>(rows_copy);
  const int hv = h / 8;
#define PULL(V, KM)                                                                      \
  combine_pull_kernel<V, KM><<<warp_grid(T), 256, 0, st>>>(peers, T, K, hv, topk_idx, inv_c, \
                                                          base, el, weights, r, x1, x2, o, cp)
  if (K <= 2)
    PULL(4, 2);
  else if (K <= 4)
    PULL(4, 4);
  else if (K <= 8)
    PULL(2, 8);
  else if (K <= 16)
    PULL(1, 16);
  else
    PULL(1, 32);
#undef PULL
  MOE_LAUNCH_CHECK();
  return kOk;
}

static int combine_bwd_push_impl(const void* dy, const void* o_local,
                                 const unsigned long long* d_peers, int T, int K, int h,
                                 const int* topk_idx, const int* inv_c, const int* base, int el,
                                 const float* prob, float* dprob, int dest, void* stream) {
  if (h % 8 || el < 1 || K > 32) return kErrInvalidArg;
  if (T == 0) return kOk;
  auto st = static_cast<cudaStream_t>(stream);
  const auto* y = static_cast<const int4*>(dy);
  const auto* ol = static_cast<const int4*>(o_local);
  const int hv = h / 8;
  if (dest >= 0) {
    // runs concurrently with the persistent GEMM that waits for it (moe_gg_fc2_dgrad_ep)
    const long long nb = ceil_div_ll(T, 4), cap = (long long)sms() * 16;
    combine_bwd_push_sel_kernel<2><<<(int)(nb < cap ? nb : cap), 128, 0, st>>>(
        y, ol, d_peers, T, K, hv, topk_idx, inv_c, base, el, prob, dprob, dest);
    MOE_LAUNCH_CHECK();
    return kOk;
  }
  const int grid = warp_grid(T), threads = 256;
#define PUSH(V, KM)                                                                        \
  combine_bwd_push_kernel<V, KM><<<grid, threads, 0, st>>>(y, ol, d_peers, T, K, hv,         \
                                                          topk_idx, inv_c, base, el, prob,     \
                                                          dprob, dest)
  if (K <= 2)
    PUSH(4, 2);
  else if (K <= 4)
    PUSH(4, 4);
  else if (K <= 8)
    PUSH(2, 8);
  else if (K <= 16)
    PUSH(1, 16);
  else
    PUSH(1, 32);
#undef PUSH
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_ep_combine_bwd_push(const void* dy, const void* o_local,
                            const unsigned long long* d_peers, int T, int K, int h,
                            const int* topk_idx, const int* inv_c, const int* base, int el,
                            const float* prob, float* dprob, void* stream) {
  return combine_bwd_push_impl(dy, o_local, d_peers, T, K, h, topk_idx, inv_c, base, el, prob,
                               dprob, -1, stream);
}

// Combine backward restricted to the selections whose expert lives on rank `dest`; dprob is
// written for those selections only.
int moe_ep_combine_bwd_push_dest(const void* dy, const void* o_local,
                                 const unsigned long long* d_peers, int T, int K, int h,
                                 const int* topk_idx, const int* inv_c, const int* base, int el,
                                 const float* prob, float* dprob, int dest, void* stream) {
  if (dest < 0) return kErrInvalidArg;
  return combine_bwd_push_impl(dy, o_local, d_peers, T, K, h, topk_idx, inv_c, base, el, prob,
                               dprob, dest, stream);
}

int moe_ep_token_ranks(const int* topk_idx, const int* inv_c, int T, int K, int el,
                       int* rank_idx, int* sel_j, int* sel_pos, void* stream) {
  if (el < 1 || K < 1) return kErrInvalidArg;
  if (T == 0) return kOk;
  token_ranks_kernel<<<ceil_div_i(T, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      topk_idx, inv_c, T, K, el, rank_idx, sel_j, sel_pos);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_ep_dispatch_dedup(const void* x, int T, int K, int h, const int* topk_idx,
                          const int* inv_c, const int* base, int el, const int* rank_idx,
                          const int* inv_rank, const int* tbase, const int* sel_j,
                          const int* sel_pos, const float* prob,
                          const unsigned long long* tok_peers,
                          const unsigned long long* map_peers,
                          const unsigned long long* srows_peers,
                          const unsigned long long* sprob_peers,
                          const unsigned long long* rprob_peers, void* stream) {
  if (h % 8 || el < 1) return kErrInvalidArg;
  if (T == 0) return kOk;
  dispatch_dedup_kernel<4><<<warp_grid(T), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(x), T, K, h / 8, topk_idx, inv_c, base, el, rank_idx, inv_rank,
      tbase, sel_j, sel_pos, prob, tok_peers, map_peers, srows_peers, sprob_peers,
      rprob_peers);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_ep_echo_rewrite(const int* topk_idx, const int* inv_c, int T, int K, int ns,
                        const int* gbase, const int* seg_start, const int* seg_v, int* topk_v,
                        void* stream) {
  const long long n = (long long)T * K;
  if (ns < 1) return kErrInvalidArg;
  if (n == 0) return kOk;
  echo_rewrite_kernel<<<(int)ceil_div_ll(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      topk_idx, inv_c, n, ns, gbase, seg_start, seg_v, topk_v);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_ep_fill_pad_map(const int* map_pad, int rows, int* map, void* stream) {
  if (rows <= 0) return kOk;
  const int blocks = ceil_div_i(rows, 256) < sms() * 4 ? ceil_div_i(rows, 256) : sms() * 4;
  fill_pad_map_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(map_pad, rows,
                                                                             map);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_ep_expand_grad(const void* tok, const int* map, int rows, int h, const float* rowprob,
                       const void* o, void* d_o, float* dprob_rows, void* stream) {
  if (h % 8) return kErrInvalidArg;
  if (rows <= 0) return kOk;
  expand_grad_kernel<<<warp_grid(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(tok), map, rows, h / 8, rowprob, static_cast<const int4*>(o),
      static_cast<int4*>(d_o), dprob_rows);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_ep_dprob_pull(const unsigned long long* part_peers, int T, int K, const int* topk_idx,
                      const int* inv_c, const int* base, int el, int ldp, float* dprob,
                      void* stream) {
  const long long n = (long long)T * K;
  if (n == 0) return kOk;
  dprob_pull_kernel<<<(int)ceil_div_ll(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      part_peers, n, K, topk_idx, inv_c, base, el, ldp, dprob);
  MOE_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"
