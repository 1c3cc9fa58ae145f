// lattice.cu -- device lattice CSR (node -> incident struts) and the degree-bucketed
// node schedule.
//
// PAPER.md Sec. 4.3.1: the auxiliary planes are precomputed "using the GPU and the
// lattice's topology graph (i.e., an adjacency list in the GPU)"; Sec. 4.3.3: workloads
// are sorted so that combinable work lands in the same warp.  Here the workload of a
// node is its degree; nodes are counting-sorted into degree buckets, each bucket served
// by a kernel instantiation sized for it (lane-group width, shared-memory capacities).
#include "lmm_internal.h"

namespace {

__global__ void k_pack_nodes(const float *xyz, int64_t N, float4 *node) {
  int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= N) return;
  node[n] = make_float4(xyz[3 * n], xyz[3 * n + 1], xyz[3 * n + 2], __int_as_float(0x7fc00000));
}

__global__ void k_pack_ends(const int64_t *ends, int64_t S, int64_t N, int2 *e32, int *deg, int *bad) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S) return;
  int64_t a = ends[2 * s], b = ends[2 * s + 1];
  if (a < 0 || b < 0 || a >= N || b >= N || a == b) { atomicAdd(bad, 1); a = b = 0; e32[s] = make_int2(-1, -1); return; }
  e32[s] = make_int2((int)a, (int)b);
  atomicAdd(&deg[a], 1);
  atomicAdd(&deg[b], 1);
}

__global__ void k_scatter_r(const int2 *e32, const float *r_end, int64_t S, float4 *node) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S) return;
  int2 e = e32[s];
  if (e.x < 0) return;
  node[e.x].w = r_end[2 * s];
  node[e.y].w = r_end[2 * s + 1];
}

// every strut end at a node must carry the node's sphere radius (struts are tangent to
// the nodal spheres, Sec. 4.1)
__global__ void k_check_r(const int2 *e32, const float *r_end, int64_t S, const float4 *node, int *bad) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S) return;
  int2 e = e32[s];
  if (e.x < 0) return;
  float r0 = r_end[2 * s], r1 = r_end[2 * s + 1];
  if (!(r0 > 0.0f) || !(r1 > 0.0f) || r0 != node[e.x].w || r1 != node[e.y].w) atomicAdd(bad, 1);
}

__global__ void k_fill(const int2 *e32, int64_t S, const int *off, int *cursor, int2 *ent) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S) return;
  int2 e = e32[s];
  int p0 = off[e.x] + atomicAdd(&cursor[e.x], 1);
  ent[p0] = make_int2((int)s, e.y);
  int p1 = off[e.y] + atomicAdd(&cursor[e.y], 1);
  ent[p1] = make_int2((int)s, (int)((unsigned)e.x | 0x80000000u));
}

// ascending strut id within each node (deterministic local side numbering): every entry is
// placed at its rank among its node's entries (thread per entry; the segment is read from
// L1), and the strut's CSR positions are recorded on the way
__global__ void k_rank_segments(const int *off, const int2 *e32, int64_t S2, const int2 *in, int2 *out, int2 *strut_csr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= S2) return;
  const int2 x = in[i];
  const bool endB = ((unsigned)x.y >> 31) != 0;
  const int2 e = e32[x.x];
  const int n = endB ? e.y : e.x;
  const int b = off[n], en = off[n + 1];
  int rank = 0;
  for (int j = b; j < en; j++) rank += __ldg(&in[j].x) < x.x ? 1 : 0;
  const int p = b + rank;
  out[p] = x;
  if (endB) strut_csr[x.x].y = p;
  else strut_csr[x.x].x = p;
}

__global__ void k_deg_hist(const int *off, int64_t N, unsigned long long *hist) {
  __shared__ unsigned int h[33];
  if (threadIdx.x < 33) h[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x) {
    int d = off[n + 1] - off[n];
    atomicAdd(&h[d > 31 ? 32 : d], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 33 && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

__host__ __device__ __forceinline__ int bucket_of(int d) {
  return d == 0 || d > LMM_MAXD ? -1 : (d <= 4 ? 0 : (d <= 8 ? 1 : (d <= 12 ? 2 : (d <= 16 ? 3 : (d <= 23 ? 4 : 5)))));
}

__global__ void k_bucket_fill(const int *off, int64_t N, const int *bucket_base, int *cursor, int *list) {
  int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= N) return;
  int b = bucket_of(off[n + 1] - off[n]);
  if (b < 0) return;
  // warp-aggregated slot claim per bucket keeps nodes of a warp contiguous
  unsigned act = __activemask();
  for (int bb = 0; bb < LMM_NBUCKET; bb++) {
    unsigned m = __match_any_sync(act, b == bb ? bb : -1 - (int)threadIdx.x);
    if (b != bb) continue;
    int leader = __ffs(m) - 1;
    int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == leader) base = atomicAdd(&cursor[bb], __popc(m));
    base = __shfl_sync(m, base, leader);
    list[bucket_base[bb] + base + __popc(m & ((1u << lane) - 1u))] = (int)n;
  }
}

__global__ void k_narrow(const int64_t *in, int64_t n, int *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i <= n) out[i] = (int)in[i];
}

}  // namespace

int lattice_build(lmm_ctx *c, const float *xyz, const int64_t *ends, const float *rend) {
  const int64_t N = c->N, S = c->S;
  int rc;
  if ((rc = dev_alloc(c->node, sizeof(float4) * (N + 1)))) return rc;
  if ((rc = dev_alloc(c->ends, sizeof(int2) * (S + 1)))) return rc;
  if ((rc = dev_alloc(c->csr_off, sizeof(int) * (N + 1)))) return rc;
  if ((rc = dev_alloc(c->csr_ent, sizeof(int2) * (2 * S + 1)))) return rc;
  if ((rc = dev_alloc(c->strut_csr, sizeof(int2) * (S + 1)))) return rc;
  if ((rc = dev_alloc(c->scratch, sizeof(int) * (N + 8) > 64 ? sizeof(int) * (N + 8) : 64))) return rc;
  int *deg = (int *)c->scratch.p;   // [N] degree then cursor, [N..N+1] bad flags
  int *bad = deg + N;
  KTimer t(c, LMM_K_CSR);
  CUDA_TRY(cudaMemsetAsync(c->scratch.p, 0, sizeof(int) * (N + 8), c->stream));
  const int T = 256;
  if (N) (c->n_launch++), k_pack_nodes<<<(unsigned)((N + T - 1) / T), T, 0, c->stream>>>(xyz, N, (float4 *)c->node.p);
  if (S) (c->n_launch++), k_pack_ends<<<(unsigned)((S + T - 1) / T), T, 0, c->stream>>>(ends, S, N, (int2 *)c->ends.p, deg, bad);
  if (S) (c->n_launch++), k_scatter_r<<<(unsigned)((S + T - 1) / T), T, 0, c->stream>>>((const int2 *)c->ends.p, rend, S, (float4 *)c->node.p);
  if (S) (c->n_launch++), k_check_r<<<(unsigned)((S + T - 1) / T), T, 0, c->stream>>>((const int2 *)c->ends.p, rend, S, (const float4 *)c->node.p, bad + 1);
  CUDA_TRY(cudaGetLastError());
  if (!c->pinned_scalar) CUDA_TRY(cudaMallocHost((void **)&c->pinned_scalar, 64));
  int *hbad = (int *)(c->pinned_scalar + 4);
  CUDA_TRY(cudaMemcpyAsync(hbad, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (hbad[0]) return LMM_E_ARG;
  if (hbad[1]) return LMM_E_RADIUS;
  // CSR offsets: exclusive scan of degrees (int32, 2S < 2^31)
  if ((rc = dev_alloc(c->tmp64, sizeof(int64_t) * (N + 2)))) return rc;
  int64_t total = 0;
  if ((rc = scan_exclusive_i32_to_i64(c, deg, (int64_t *)c->tmp64.p, N, &total))) return rc;
  if (total != 2 * S) return LMM_E_ARG;
  (c->n_launch++), k_narrow<<<(unsigned)((N + 1 + T - 1) / T), T, 0, c->stream>>>((const int64_t *)c->tmp64.p, N, (int *)c->csr_off.p);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemsetAsync(deg, 0, sizeof(int) * N, c->stream));
  if (S) (c->n_launch++), k_fill<<<(unsigned)((S + T - 1) / T), T, 0, c->stream>>>((const int2 *)c->ends.p, S, (const int *)c->csr_off.p, deg, (int2 *)c->csr_ent.p);
  if (S) {
    if ((rc = dev_alloc(c->csr_tmp, sizeof(int2) * (2 * S + 1)))) return rc;
    (c->n_launch++), k_rank_segments<<<(unsigned)((2 * S + T - 1) / T), T, 0, c->stream>>>(
        (const int *)c->csr_off.p, (const int2 *)c->ends.p, 2 * S, (const int2 *)c->csr_ent.p, (int2 *)c->csr_tmp.p,
        (int2 *)c->strut_csr.p);
    DevBuf t = c->csr_ent;   // the ranked copy becomes the CSR
    c->csr_ent = c->csr_tmp;
    c->csr_tmp = t;
  }
  CUDA_TRY(cudaGetLastError());
  return LMM_OK;
}

int degree_buckets(lmm_ctx *c) {
  const int64_t N = c->N;
  int rc;
  if ((rc = dev_alloc(c->deg_hist, sizeof(unsigned long long) * 33))) return rc;
  if ((rc = dev_alloc(c->bucket_nodes, sizeof(int) * (N + 1)))) return rc;
  if ((rc = dev_alloc(c->bucket_cnt, sizeof(int) * 16))) return rc;
  KTimer t(c, LMM_K_BUCKET);
  CUDA_TRY(cudaMemsetAsync(c->deg_hist.p, 0, sizeof(unsigned long long) * 33, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->bucket_cnt.p, 0, sizeof(int) * 16, c->stream));
  const int T = 256;
  if (N) {
    int grid = (int)((N + T - 1) / T);
    if (grid > c->n_sm * 8) grid = c->n_sm * 8;
    (c->n_launch++), k_deg_hist<<<grid, T, 0, c->stream>>>((const int *)c->csr_off.p, N, (unsigned long long *)c->deg_hist.p);
  }
  if (!c->pinned_hist) CUDA_TRY(cudaMallocHost((void **)&c->pinned_hist, 64 * sizeof(unsigned long long)));
  unsigned long long *h = c->pinned_hist;
  CUDA_TRY(cudaMemcpyAsync(h, c->deg_hist.p, 33 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  int64_t cnt[LMM_NBUCKET] = {0};
  for (int d = 1; d <= 31; d++) cnt[bucket_of(d)] += (int64_t)h[d];
  c->bucket_off[0] = 0;
  for (int b = 0; b < LMM_NBUCKET; b++) c->bucket_off[b + 1] = c->bucket_off[b] + cnt[b];
  int *base = (int *)(c->pinned_hist + 40);
  for (int b = 0; b < LMM_NBUCKET; b++) base[b] = (int)c->bucket_off[b];
  int *dbase = (int *)c->bucket_cnt.p + 8;
  CUDA_TRY(cudaMemcpyAsync(dbase, base, LMM_NBUCKET * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  if (N) (c->n_launch++), k_bucket_fill<<<(unsigned)((N + T - 1) / T), T, 0, c->stream>>>((const int *)c->csr_off.p, N, dbase, (int *)c->bucket_cnt.p, (int *)c->bucket_nodes.p);
  CUDA_TRY(cudaGetLastError());
  return LMM_OK;
}
