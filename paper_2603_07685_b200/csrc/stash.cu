// Paged Stashing (reference allocator pkg/src/moelab/planners.py:394-463)
// as device-initiated kernels, so a multi-layer sync-free step stays CUDA-graph capturable.
//
// The layer's saved activations live in ONE worst-case "tmp" buffer set shared by all layers;
// after a layer's forward its ACTUAL rows (a device count, e.g. the plan's rows_pad) are
// copied into fixed-size pages taken from the head of a circular free list, and before its
// backward they are copied back and the pages returned to the tail. Memory is
// O(worst_case + sum(actual)) instead of O(layers x worst_case).
//
// state[0] head, [1] free pages, [2] peak pages in use, [3] failed stashes (sticky),
// [4] result of the last allocation (0 ok, 1 out of pages).
// record[0] = pages held (-1: the stash failed), record[1..] = page ids in order.
#include "common.cuh"

namespace moe {
namespace stash {

__global__ void init_kernel(int* state, int* ring, int num_pages) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < num_pages; i += gridDim.x * blockDim.x)
    ring[i] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[0] = 0;
    state[1] = num_pages;
    state[2] = 0;
    state[3] = 0;
    state[4] = 0;
  }
}

__global__ void alloc_kernel(int* state, const int* ring, int num_pages, int page_rows,
                             const int* rows_dev, int rows_host, int* record, int max_pages) {
  const int tokens = rows_dev ? *rows_dev : rows_host;
  const int need = (tokens + page_rows - 1) / page_rows;
  const int head = state[0], free_pages = state[1];
  if (need > free_pages || need > max_pages) {  // planners.py:441-446 "out of pages"
    record[0] = -1;
    state[3] += 1;
    state[4] = 1;
    return;
  }
  for (int i = 0; i < need; ++i) record[1 + i] = ring[(head + i) % num_pages];
  record[0] = need;
  state[0] = (head + need) % num_pages;
  state[1] = free_pages - need;
  const int used = num_pages - state[1];
  if (used > state[2]) state[2] = used;
  state[4] = 0;
}

__global__ void release_kernel(int* state, int* ring, int num_pages, int* record) {
  const int n = record[0];
  if (n <= 0) return;
  const int tail = (state[0] + state[1]) % num_pages;
  for (int i = 0; i < n; ++i) ring[(tail + i) % num_pages] = record[1 + i];
  state[1] += n;
  record[0] = 0;
}

// rows [0, rows) of a dense [*, row_bytes] buffer (row stride ld_bytes) <-> the record's pages.
__global__ void copy_kernel(uint8_t* dense, long long ld_bytes, uint8_t* pool, int page_rows,
                            long long row_bytes, const int* record, const int* rows_dev,
                            int rows_host, int max_rows, int to_pages) {
  int rows = rows_dev ? *rows_dev : rows_host;
  rows = rows < max_rows ? rows : max_rows;
  const int vpr = static_cast<int>(row_bytes / 16);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  if (record[0] < 0) {
    // failed stash (out of pages, planners.py:441-446 MemoryError): nothing was recorded.
    // The reload poisons the destination rows with all-ones bytes (bf16 / fp32 NaN, int
    // -1) so the backward cannot silently compute on another layer's activations; the
    // sticky state[3] makes PagedStashBuffer.check() raise MemoryError.
    if (!to_pages)
      for (int r = warp; r < rows; r += nwarps) {
        int4* d = reinterpret_cast<int4*>(dense + (long long)r * ld_bytes);
        for (int c = lane; c < vpr; c += 32) d[c] = make_int4(-1, -1, -1, -1);
      }
    return;
  }
  for (int r = warp; r < rows; r += nwarps) {
    const int page = __ldg(record + 1 + r / page_rows);
    int4* p = reinterpret_cast<int4*>(pool + ((long long)page * page_rows + r % page_rows) *
                                                 row_bytes);
    int4* d = reinterpret_cast<int4*>(dense + (long long)r * ld_bytes);
    if (to_pages) {
      for (int c = lane; c < vpr; c += 32) st_na_v4(p + c, ld_nc_v4(d + c));
    } else {
      for (int c = lane; c < vpr; c += 32) d[c] = ld_nc_v4(p + c);
    }
  }
}

static int sms() { return device_sms(); }

}  // namespace stash
}  // namespace moe

using namespace moe;

extern "C" {

int moe_stash_init(int* state, int* ring, int num_pages, void* stream) {
  if (num_pages < 1) return kErrInvalidArg;
  const int g = ceil_div_i(num_pages, 256) < 1024 ? ceil_div_i(num_pages, 256) : 1024;
  stash::init_kernel<<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(state, ring, num_pages);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_stash_alloc(int* state, const int* ring, int num_pages, int page_rows,
                    const int* rows_dev, int rows_host, int* record, int max_pages,
                    void* stream) {
  if (num_pages < 1 || page_rows < 1 || max_pages < 0) return kErrInvalidArg;
  stash::alloc_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      state, ring, num_pages, page_rows, rows_dev, rows_host, record, max_pages);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_stash_release(int* state, int* ring, int num_pages, int* record, void* stream) {
  if (num_pages < 1) return kErrInvalidArg;
  stash::release_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(state, ring, num_pages,
                                                                        record);
  MOE_LAUNCH_CHECK();
  return kOk;
}

int moe_stash_copy(void* dense, long long ld_bytes, void* pool, int page_rows,
                   long long row_bytes, const int* record, const int* rows_dev, int rows_host,
                   int max_rows, int to_pages, void* stream) {
  if (page_rows < 1 || row_bytes <= 0 || (row_bytes & 15) || (ld_bytes & 15) ||
      (reinterpret_cast<uintptr_t>(dense) & 15) || (reinterpret_cast<uintptr_t>(pool) & 15))
    return kErrInvalidArg;
  if (max_rows <= 0) return kOk;
  const int g = ceil_div_i(max_rows, 8) < stash::sms() * 8 ? ceil_div_i(max_rows, 8)
                                                           : stash::sms() * 8;
  stash::copy_kernel<<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(dense), ld_bytes, static_cast<uint8_t*>(pool), page_rows, row_bytes,
      record, rows_dev, rows_host, max_rows, to_pages);
  MOE_LAUNCH_CHECK();
  return kOk;
}

}  // extern "C"
