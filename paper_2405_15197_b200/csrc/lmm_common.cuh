// lmm_common.cuh -- device-side definitions shared by the liblmm kernels.
//
// Binary32 arithmetic in the meta-mesh and decision paths follows the fixed-order
// specification of DESIGN.md Sec. 4 (the kernels are compiled with -fmad=false so no
// multiply-add is contracted; '/' and sqrtf are IEEE round-to-nearest).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/lmm.h"

#define LMM_MAXD 31         // degree-bucketed kernels (metamesh.cu): sides 0..31 in 32-bit masks
#define LMM_MAXD_SPILL 63   // spill kernel (spill.cu): sides 0..63 in 64-bit masks
#define LMM_NODE_SPILL 0xfe // internal node status: left for the spill kernel (never reported)
#define LMM_MAX_LEVEL 4     // vertex resolution delta_c 2^level, level 0..4 (reading R10)
#define LMM_TOL_REL 1e-4f   // delta   = TOL * R  : tie tolerance
#define LMM_CTOL_REL 1e-3f  // delta_c = CTOL * R : vertex clustering radius
#define LMM_PI_F 3.14159265358979324f
#define LMM_TWO_PI_F 6.28318530717958648f
#define LMM_HALF_PI_F 1.57079632679489662f

// ---------------------------------------------------------------------------------
// per-node slabs: capacity is a linear function of the degree d so that the slab base
// of node n is K * csr_off[n] + K0 * n (no extra scan).  DESIGN.md Sec. 5.
// ---------------------------------------------------------------------------------
#define SLAB_V_K 2      // vertices      <= 2d + 2
#define SLAB_V_K0 2
#define SLAB_A_K 3      // arcs          <= 3d + 2
#define SLAB_A_K0 2
#define SLAB_L_K 6      // loop entries  <= 6d + 4
#define SLAB_L_K0 4
#define SLAB_H_K 2      // holes         <= 2d + 2
#define SLAB_H_K0 2
#define SLAB_HE_K 3     // hole entries  <= 3d + 2
#define SLAB_HE_K0 2

__host__ __device__ inline int64_t slab_base(int64_t off_n, int64_t n, int k, int k0) { return k * off_n + k0 * n; }
__host__ __device__ inline int slab_cap(int d, int k, int k0) { return k * d + k0; }

// arc record: 12 x 32 bit (48 B)
struct ArcRec {
  uint32_t ids;   // lo | hi<<6 | vs<<12 | ve<<22 (arc_ids): sides 0..63, vertex ids 0..1023
  float t0, dt;
  float ox, oy, oz, ax, ay, az, bx, by, bz;
};
static_assert(sizeof(ArcRec) == 48, "arc record is 48 bytes");
// arc sides (lo < hi, 0 = sphere) and end vertices packed in ArcRec.ids
__host__ __device__ __forceinline__ uint32_t arc_ids(int lo, int hi, int vs, int ve) {
  return (uint32_t)lo | ((uint32_t)hi << 6) | ((uint32_t)vs << 12) | ((uint32_t)ve << 22);
}
__host__ __device__ __forceinline__ int arc_lo(uint32_t i) { return (int)(i & 63u); }
__host__ __device__ __forceinline__ int arc_hi(uint32_t i) { return (int)((i >> 6) & 63u); }
__host__ __device__ __forceinline__ int arc_vs(uint32_t i) { return (int)((i >> 12) & 1023u); }
__host__ __device__ __forceinline__ int arc_ve(uint32_t i) { return (int)(i >> 22); }

// loop entry: arc | fwd<<16, phs, dph, cum (first point index within the loop)
struct LoopRec {
  uint32_t arc_fwd;
  float phs, dph;
  int32_t cum;   // point offset in the ring (count pass, low 22 bits) | start vertex << 22 (meta-mesh)
};
#define LE_VID_SHIFT 22
#define LE_CUM_MASK 0x3fffff
#define LE_VID_MASK ((int32_t)0xffc00000)
__host__ __device__ inline int le_cum(int32_t c) { return c & LE_CUM_MASK; }
__host__ __device__ inline int le_vid(int32_t c) { return (int)((uint32_t)c >> LE_VID_SHIFT); }
static_assert(sizeof(LoopRec) == 16, "loop record is 16 bytes");

// hole entry: arc | fwd<<16, cum
struct HoleEnt {
  uint32_t arc_fwd;
  int32_t cum;
};

// ---------------------------------------------------------------------------------
// binary32 vector helpers (operation order as in DESIGN.md Sec. 4)
// ---------------------------------------------------------------------------------
struct f3 { float x, y, z; };
__device__ __forceinline__ f3 F3(float x, float y, float z) { f3 r; r.x = x; r.y = y; r.z = z; return r; }
__device__ __forceinline__ f3 f_sub(f3 a, f3 b) { return F3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ f3 f_add(f3 a, f3 b) { return F3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ f3 f_scl(f3 a, float s) { return F3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ f3 f_div(f3 a, float s) { return F3(a.x / s, a.y / s, a.z / s); }
// dot and cross products with explicit fused multiply-adds
__device__ __forceinline__ float f_dot(f3 a, f3 b) { return __fmaf_rn(a.z, b.z, __fmaf_rn(a.y, b.y, __fmul_rn(a.x, b.x))); }
__device__ __forceinline__ f3 f_cross(f3 a, f3 b) {
  return F3(__fmaf_rn(a.y, b.z, -__fmul_rn(a.z, b.y)), __fmaf_rn(a.z, b.x, -__fmul_rn(a.x, b.z)),
            __fmaf_rn(a.x, b.y, -__fmul_rn(a.y, b.x)));
}
__device__ __forceinline__ f3 f_nrm(f3 a) { return f_div(a, sqrtf(f_dot(a, a))); }

// Four-quadrant arc tangent with + - * / only: bit-identical across implementations
// that evaluate the same operations.
__device__ __forceinline__ float atan2p(float y, float x) {
  float ax = fabsf(x), ay = fabsf(y);
  float mx = ax > ay ? ax : ay;
  float mn = ax > ay ? ay : ax;
  if (mx == 0.0f) return 0.0f;
  float r = mn / mx;
  float y0 = 0.0f;
  if (r > 0.41421356237309503f) { y0 = 0.78539816339744831f; r = (r - 1.0f) / (r + 1.0f); }
  float z = r * r;
  float p = ((8.05374449538e-2f * z - 1.38776856032e-1f) * z + 1.99777106478e-1f) * z - 3.33329491539e-1f;
  float a = y0 + (p * z * r + r);
  if (ay > ax) a = LMM_HALF_PI_F - a;
  if (x < 0.0f) a = LMM_PI_F - a;
  if (y < 0.0f) a = -a;
  return a;
}
