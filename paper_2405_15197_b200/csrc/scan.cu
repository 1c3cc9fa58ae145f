// scan.cu -- device exclusive prefix scan (int32 or int64 in, int64 out).
//
// PAPER.md Sec. 4.3.2: "the prefix-sum array in the index region can be efficiently
// obtained in GPU through parallel scanning algorithms".  Reduce-then-scan: tile sums,
// a recursive scan of the tile sums, then a per-tile scan with the tile's offset.  Tiles
// of 2048 elements (256 threads x 8), warp shuffles inside the tile.
#include "lmm_internal.h"

namespace {

constexpr int SCAN_T = 256;
constexpr int SCAN_V = 8;
constexpr int SCAN_TILE = SCAN_T * SCAN_V;

template <class T> __device__ __forceinline__ int64_t ld(const T *p, int64_t i, int64_t n) { return i < n ? (int64_t)p[i] : 0; }

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *total) {
  __shared__ int64_t wsum[SCAN_T / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < SCAN_T / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < SCAN_T / 32) wsum[lane] = w;
  }
  __syncthreads();
  int64_t wpre = wid ? wsum[wid - 1] : 0;
  *total = wsum[SCAN_T / 32 - 1];
  __syncthreads();
  return wpre + x - v;
}

template <class T> __global__ void k_tile_sums(const T *in, int64_t n, int64_t *sums) {
  int64_t base = blockIdx.x * (int64_t)SCAN_TILE + threadIdx.x * SCAN_V;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_V; i++) s += ld(in, base + i, n);
  int64_t tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <class T> __global__ void k_tile_scan(const T *in, int64_t n, const int64_t *tile_off, int64_t *out) {
  int64_t base = blockIdx.x * (int64_t)SCAN_TILE + threadIdx.x * SCAN_V;
  int64_t v[SCAN_V];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_V; i++) { v[i] = ld(in, base + i, n); s += v[i]; }
  int64_t tot;
  int64_t pre = block_excl_scan(s, &tot) + (tile_off ? tile_off[blockIdx.x] : 0);
#pragma unroll
  for (int i = 0; i < SCAN_V; i++) {
    if (base + i <= n) out[base + i] = pre;   // out[n] = grand total
    pre += v[i];
  }
}

// scratch for the tile sums of every recursion level, grown once (no per-call
// allocation: stream-ordered allocation inside a timed step stalls the host)
static size_t scan_scratch_elems(int64_t n) {
  size_t tot = 0;
  int64_t m = n;
  while (true) {
    int64_t nt = (m + 1 + SCAN_TILE - 1) / SCAN_TILE;
    if (nt <= 1) break;
    tot += 2 * (size_t)nt + 2;
    m = nt;
  }
  return tot + 2;
}

template <class T> int scan_impl(lmm_ctx *c, const T *in, int64_t *out, int64_t n, int64_t *scratch) {
  // out has n+1 entries; out[n] = total
  int64_t ntile = (n + 1 + SCAN_TILE - 1) / SCAN_TILE;
  if (ntile <= 1) {
    (c->n_launch++), k_tile_scan<T><<<1, SCAN_T, 0, c->stream>>>(in, n, nullptr, out);
  } else {
    int64_t *sums = scratch, *soff = scratch + ntile + 1;
    (c->n_launch++), k_tile_sums<T><<<(unsigned)ntile, SCAN_T, 0, c->stream>>>(in, n, sums);
    CUDA_TRY(cudaGetLastError());
    int rc = scan_impl<int64_t>(c, sums, soff, ntile, scratch + 2 * ntile + 2);
    if (rc) return rc;
    (c->n_launch++), k_tile_scan<T><<<(unsigned)ntile, SCAN_T, 0, c->stream>>>(in, n, soff, out);
  }
  CUDA_TRY(cudaGetLastError());
  return LMM_OK;
}

template <class T> int scan_top(lmm_ctx *c, const T *in, int64_t *out, int64_t n, int64_t *total_host) {
  int rc;
  if ((rc = dev_alloc(c->scan_tmp, sizeof(int64_t) * scan_scratch_elems(n)))) return rc;
  if (!c->pinned_scalar) CUDA_TRY(cudaMallocHost((void **)&c->pinned_scalar, 64));
  if ((rc = scan_impl<T>(c, in, out, n, (int64_t *)c->scan_tmp.p))) return rc;
  if (total_host) {
    CUDA_TRY(cudaMemcpyAsync(c->pinned_scalar, out + n, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    *total_host = c->pinned_scalar[0];
  }
  return LMM_OK;
}

}  // namespace

int scan_exclusive_i64(lmm_ctx *c, const int64_t *in, int64_t *out, int64_t n, int64_t *total_host) {
  KTimer t(c, LMM_K_SCAN);
  return scan_top<int64_t>(c, in, out, n, total_host);
}

int scan_exclusive_i32_to_i64(lmm_ctx *c, const int *in, int64_t *out, int64_t n, int64_t *total_host) {
  KTimer t(c, LMM_K_SCAN);
  return scan_top<int>(c, in, out, n, total_host);
}
