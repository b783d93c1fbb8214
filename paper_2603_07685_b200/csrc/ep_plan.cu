// Device-side EP exchange plan: the sync-free replacement of the host planning that follows
// the counts all-gather (dispatcher.ep_host_plan / p2p_tables / global_aux, which stay as the
// host restatement the tests compare against).
//
// From the all-gathered per-rank [counts | mean scores] rows it derives, on the GPU, every
// table the p2p transport needs -- so the EP forward never reads the counts on the host and
// the whole fwd+bwd step can be captured in a CUDA graph (PAPER.md
// sync-free dropless MoE):
//   * global-position capacity (apply_capacity routing.py:226-247 on the GLOBAL batch):
//     slot j of expert e on rank s is kept iff sum_{s'<s} counts[s', e] + j < C;
//   * this rank's padded plan (expert blocks aligned to `align` rows, phantom rows with pad),
//     its regroup table, 128-row block -> expert map and [blocks, rows] meta;
//   * base[e]: where this rank's compact rows of expert e land in e's home-rank plan;
//   * dst_off[s, j]: source s's compact offset of this rank's j-th expert (scatter epilogues);
//   * the global aux loss (routing.py:111-120) and its per-expert score gradient.
#include "common.cuh"

namespace moe {
namespace epplan {

__global__ void ep_plan_kernel(const float* __restrict__ g, int ldg, int n, int E, int me,
                               int T, int K, int capacity, int pad, int align, float coeff,
                               int rows_cap, int* __restrict__ base, int* __restrict__ cap_local,
                               int* __restrict__ table, int* __restrict__ block_expert,
                               int max_blocks, int* __restrict__ meta,
                               int* __restrict__ dst_off, float* __restrict__ aux,
                               float* __restrict__ aux_grad, int* __restrict__ status) {
  extern __shared__ int sm[];
  int* counts = sm;              // [n, E]
  int* kept = counts + n * E;    // [n, E]
  int* padded = kept + n * E;    // [E]
  int* offl = padded + E;        // [el + 1] this rank's padded offsets
  __shared__ float red[1024];
  const int el = E / n;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < n * E; i += nt) counts[i] = __float2int_rn(g[(i / E) * ldg + i % E]);
  __syncthreads();
  float part = 0.f;
  for (int e = tid; e < E; e += nt) {
    int prefix = 0, tot = 0, real = 0, prefix_me = 0;
    for (int s = 0; s < n; ++s) {
      const int c = counts[s * E + e];
      int k = c;
      if (capacity >= 0) k = min(max(capacity - prefix, 0), c);
      kept[s * E + e] = k;
      if (s == me) prefix_me = prefix;
      prefix += c;
      tot += c;
      real += k;
    }
    cap_local[e] = capacity >= 0 ? max(capacity - prefix_me, 0) : -1;
    const int phantom = (capacity >= 0 && pad) ? capacity - min(tot, capacity) : 0;
    const int eff = real + phantom;
    padded[e] = (eff + align - 1) / align * align;
    // aux loss (routing.py:117-119 on the global batch): f = counts / (n T K), P = mean score
    const float f = static_cast<float>(tot) / static_cast<float>(max(n * T * K, 1));
    float P = 0.f;
    for (int s = 0; s < n; ++s) P += g[s * ldg + E + e];
    P /= static_cast<float>(n);
    part += f * P;
    aux_grad[e] = coeff * static_cast<float>(E) * f / static_cast<float>(max(n * T, 1));
  }
  red[tid] = part;
  __syncthreads();
  for (int w = nt / 2; w > 0; w >>= 1) {  // fixed-order tree: deterministic
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  if (tid == 0) aux[0] = coeff * static_cast<float>(E) * red[0];
  if (tid == 0) {
    int a = 0;
    for (int j = 0; j < el; ++j) {
      offl[j] = a;
      a += padded[me * el + j];
    }
    offl[el] = a;
  }
  __syncthreads();
  const int rows_pad = offl[el];
  // table = [kept_mine n*el | recv_off n*el | off_pad el+1 | real el]
  int* t_kept = table;
  int* t_recv = table + n * el;
  int* t_off = t_recv + n * el;
  int* t_real = t_off + el + 1;
  for (int e = tid; e < E; e += nt) {
    const int r = e / el, j = e % el;
    int off_home = 0;
    for (int q = 0; q < j; ++q) off_home += padded[r * el + q];
    int pk = 0;
    for (int s = 0; s < me; ++s) pk += kept[s * E + e];
    int offc = 0;
    for (int q = 0; q < e; ++q) offc += kept[me * E + q];
    base[e] = off_home + pk - offc;
  }
  for (int i = tid; i < n * el; i += nt) {
    const int s = i / el, j = i % el, e = me * el + j;
    t_kept[i] = kept[s * E + e];
    int ro = 0;
    for (int s2 = 0; s2 < s; ++s2)
      for (int q = 0; q < el; ++q) ro += kept[s2 * E + me * el + q];
    for (int q = 0; q < j; ++q) ro += kept[s * E + me * el + q];
    t_recv[i] = ro;
    int d = 0;
    for (int q = 0; q < e; ++q) d += kept[s * E + q];
    dst_off[i] = d;
  }
  for (int j = tid; j <= el; j += nt) t_off[j] = offl[j];
  for (int j = tid; j < el; j += nt) {
    int rl = 0;
    for (int s = 0; s < n; ++s) rl += kept[s * E + me * el + j];
    t_real[j] = rl;
  }
  const int nblocks = rows_pad / 128;
  for (int b = tid; b < nblocks && b < max_blocks; b += nt) {
    int lo = 0, hi = el - 1;  // last j with offl[j] <= 128 b
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (offl[mid] <= b * 128) lo = mid; else hi = mid - 1;
    }
    block_expert[b] = lo;
  }
  // Consistency of the group: every rank routed T*K selections (equal T per rank: the
  // symmetric buffers and the capacity are sized from T), and no rank's plan exceeds the
  // static rows. Otherwise poison base[] (pushes / pulls skip negative rows), run no GEMM
  // block and flag the status, so nothing is written past a peer's allocation.
  __shared__ int bad;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int s = tid; s < n; s += nt) {
    long long tot = 0, rows_s = 0;
    for (int e = 0; e < E; ++e) tot += counts[s * E + e];
    for (int j = 0; j < el; ++j) rows_s += padded[s * el + j];
    if (tot != (long long)T * K || rows_s > rows_cap) atomicOr(&bad, 1);
  }
  __syncthreads();
  if (bad) {
    for (int e = tid; e < E; e += nt) base[e] = -(1 << 30);
    // and an empty local plan: no regroup rows, no scatter rows, zero-row weight gradients
    for (int i = tid; i < 2 * n * el + 2 * el + 1; i += nt) table[i] = 0;
  }
  if (tid == 0) {
    meta[0] = bad ? 0 : nblocks;  // an inconsistent / overflowing plan runs no GEMM blocks
    meta[1] = bad ? 0 : rows_pad;
    meta[2] = 0;
    if (bad && status) atomicExch(status, 1);
  }
}

}  // namespace epplan
}  // namespace moe

using namespace moe;

extern "C" int moe_ep_plan_device(const float* gathered, int ldg, int n, int E, int me, int T,
                                  int K, int capacity, int pad, int align, float coeff,
                                  int rows_cap, int* base, int* cap_local, int* table,
                                  int* block_expert, int max_blocks, int* meta, int* dst_off,
                                  float* aux, float* aux_grad, int* status, void* stream) {
  if (n < 1 || E % n || E > 1024 || me < 0 || me >= n || (align != 128 && align != 256) ||
      ldg < 2 * E)
    return kErrInvalidArg;
  const int smem = (2 * n * E + E + E / n + 1) * static_cast<int>(sizeof(int));
  if (smem > 48 * 1024)
    MOE_CUDA_CHECK(
        ensure_dyn_smem(reinterpret_cast<const void*>(epplan::ep_plan_kernel), smem));
  epplan::ep_plan_kernel<<<1, 1024, smem, static_cast<cudaStream_t>(stream)>>>(
      gathered, ldg, n, E, me, T, K, capacity, pad, align, coeff, rows_cap, base, cap_local,
      table, block_expert, max_blocks, meta, dst_off, aux, aux_grad, status);
  MOE_LAUNCH_CHECK();
  return kOk;
}
