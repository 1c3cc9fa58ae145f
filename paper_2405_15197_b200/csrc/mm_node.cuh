// mm_node.cuh -- the per-node binary32 decision arithmetic shared by the meta-mesh kernels
// (metamesh.cu: degree-bucketed lane groups; spill.cu: CTA per node for the nodes the
// buckets cannot hold).  DESIGN.md Sec. 4: every operation rounds as written (both files
// are compiled with -fmad=false), fused multiply-adds only where the specification has them.
#pragma once
#include "lmm_common.cuh"

namespace mm {

// packed fp32 pairs (sm_100 add/mul .f32x2, round-to-nearest per lane)
// (register-pair moves: no integer shifts between the packed operations)
__device__ __forceinline__ unsigned long long f2u(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 u2f(unsigned long long u) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(u));
  return r;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(r);
}
// h_m at two points at once, each lane rounded like the scalar hs(m, y) - tau: the product, two
// explicit fused multiply-adds, then + (-e) and + (-tau).  (Never write a packed add of a packed
// product: ptxas contracts add.rn.f32x2 of a mul.rn.f32x2 result into FFMA2 even under
// -fmad=false; tests/test_abi.py checks the PTX for such pairs.)
__device__ __forceinline__ float2 side_h2(float4 p0, float4 p1, float2 Yx, float2 Yy, float2 Yz, float2 nT) {
  float2 h = mul2(make_float2(p0.x, p0.y), Yx);
  h = fma2(make_float2(p0.z, p0.w), Yy, h);
  h = fma2(make_float2(p1.x, p1.y), Yz, h);
  return add2(add2(h, make_float2(p1.z, p1.w)), nT);
}

template <class WS> struct Node {
  WS &w;
  int d;
  float R;
  __device__ f3 W(int k) const { const float4 q = w.w4[k]; return F3(q.x, q.y, q.z); }
  __device__ float E(int k) const { return w.w4[k].w; }
  __device__ f3 U(int k) const { return F3(w.ux[k], w.uy[k], w.uz[k]); }
  __device__ f3 AS(int k) const { return F3(w.asx[k], w.asy[k], w.asz[k]); }
  __device__ f3 E1(int k) const { return F3(w.e1x[k], w.e1y[k], w.e1z[k]); }
  __device__ f3 E2(int k) const { return F3(w.e2x[k], w.e2y[k], w.e2z[k]); }
  __device__ f3 V(int q) const { return F3(w.vx[q], w.vy[q], w.vz[q]); }
  __device__ float h(int k, f3 y) const { return k == 0 ? 0.0f : hs(k, y); }
  // strut side k >= 1: fma(w.z, y.z, fma(w.y, y.y, w.x y.x)) - e
  __device__ float hs(int k, f3 y) const {
    const float4 q = w.w4[k];
    return __fsub_rn(f_dot(F3(q.x, q.y, q.z), y), q.w);
  }

  // triple junction (oracle junction32), without branches: the three
  // rejection tests become a flag and the divisors of rejected lanes are replaced by 1 (their
  // roots are never used), so the group stays converged; accepted lanes compute exactly the
  // specification's operations
  __device__ bool junction_bf(int a, int b, int c, f3 *y, float *tau) const {
    f3 Wa = W(a), Wb = W(b), Wc = W(c);
    float Ea = E(a), Eb = E(b), Ec = E(c);   // side 0 (the sphere) has W = 0, E = 0
    f3 n1 = f_sub(Wa, Wb), n2 = f_sub(Wa, Wc);
    float q1 = Ea - Eb, q2 = Ea - Ec;
    f3 m = f_cross(n1, n2);
    float mm = f_dot(m, m);
    float nn1 = f_dot(n1, n1), nn2 = f_dot(n2, n2);
    bool ok = mm > (1e-8f * nn1) * nn2;
    mm = ok ? mm : 1.0f;
    f3 c1 = f_cross(n2, m), c2 = f_cross(m, n1);
    float imm = 1.0f / mm;
    f3 y0 = F3(__fmaf_rn(q2, c2.x, __fmul_rn(q1, c1.x)) * imm, __fmaf_rn(q2, c2.y, __fmul_rn(q1, c1.y)) * imm,
               __fmaf_rn(q2, c2.z, __fmul_rn(q1, c1.z)) * imm);
    float iml = 1.0f / sqrtf(mm);
    f3 mh = f_scl(m, iml);
    float tau0 = f_dot(Wa, y0) - Ea;
    float tau1 = f_dot(Wa, mh);
    float A = __fmaf_rn(-tau1, tau1, 1.0f);
    ok = ok && A > 1e-6f;
    A = ok ? A : 1.0f;
    float Bp = __fmaf_rn(-tau0, tau1, f_dot(y0, mh));
    float C = __fmaf_rn(-tau0, tau0, __fmaf_rn(-R, R, f_dot(y0, y0)));
    float disc = __fmaf_rn(Bp, Bp, -__fmul_rn(A, C));
    ok = ok && !(disc < 0.0f);
    disc = ok ? disc : 0.0f;
    float sq = sqrtf(disc);
    float iA = 1.0f / A;
    float l0 = (-Bp - sq) * iA, l1 = (-Bp + sq) * iA;
    y[0] = F3(__fmaf_rn(mh.x, l0, y0.x), __fmaf_rn(mh.y, l0, y0.y), __fmaf_rn(mh.z, l0, y0.z));
    tau[0] = __fmaf_rn(l0, tau1, tau0);
    y[1] = F3(__fmaf_rn(mh.x, l1, y0.x), __fmaf_rn(mh.y, l1, y0.y), __fmaf_rn(mh.z, l1, y0.z));
    tau[1] = __fmaf_rn(l1, tau1, tau0);
    return ok;
  }

  // branch-free over the sides (same boolean as the early-exit form)
  __device__ bool valid_strut_pt(uint32_t excl, f3 y, float tau, float delta) const {
    bool ok = !(tau < -delta);
#pragma unroll 1
    for (int m = 1; m <= d; m++) {
      bool viol = hs(m, y) - tau > delta;
      ok = ok && (((excl >> m) & 1u) || !viol);
    }
    return ok;
  }
  // both roots of a triple junction in one pass over the sides: strut junctions
  // (valid_strut_pt) or, for a sphere triple (tau taken as 0; h - 0 == h exactly), the
  // tolerant sphere-junction test "no other strut above the sphere by more than delta".
  // The two roots go through packed f32x2 operations: every lane of those rounds like the
  // scalar op (same bits as hs(m, y) - tau), h - e as h + (-e), h - tau as h + (-tau).
  __device__ void valid_junction_pair(bool sphere, uint32_t excl, f3 y0, float t0, f3 y1, float t1, float delta,
                                      bool *ok0, bool *ok1) const {
    bool k0 = *ok0 && (sphere || !(t0 < -delta)), k1 = *ok1 && (sphere || !(t1 < -delta));
    if (sphere) { t0 = 0.0f; t1 = 0.0f; }
    const float2 Yx = make_float2(y0.x, y1.x), Yy = make_float2(y0.y, y1.y), Yz = make_float2(y0.z, y1.z);
    const float2 nT = make_float2(-t0, -t1);
    uint32_t v0 = 0u, v1 = 0u, mb = 2u;   // sides violated by each root (bit m)
    for (int m = 1; m <= d; m++, mb <<= 1) {
      const float4 p0 = w.wp[m][0], p1 = w.wp[m][1];
      const float2 h = side_h2(p0, p1, Yx, Yy, Yz, nT);
      v0 |= h.x > delta ? mb : 0u;
      v1 |= h.y > delta ? mb : 0u;
    }
    *ok0 = k0 && !(v0 & ~excl); *ok1 = k1 && !(v1 & ~excl);
  }
  // end-circle (cap) point: strictly exposed
  __device__ bool valid_sphere_pt(uint32_t excl, f3 y, float delta) const {
    bool ok = true;
#pragma unroll 1
    for (int m = 1; m <= d; m++) ok = ok && (((excl >> m) & 1u) || !(hs(m, y) > -delta));
    return ok;
  }

  // PAPER.md Eq. 7: strut a's ellipse in the auxiliary plane P_{a,b}
  __device__ bool ellipse(int a, int b, f3 *o, f3 *av, f3 *bv) const {
    f3 N = f_sub(W(a), W(b));
    float inl = 1.0f / sqrtf(f_dot(N, N));
    f3 n = f_scl(N, inl);
    float pc = (E(a) - E(b)) * inl;
    f3 p = f_scl(n, pc);
    float s = w.s[a], c = w.c[a];
    f3 u = U(a);
    if (!(fabsf(f_dot(n, u)) > fabsf(s) + 1e-3f)) return false;
    f3 dd = F3(-u.x, -u.y, -u.z);
    f3 dp = f_cross(dd, n);
    float dpl2 = f_dot(dp, dp);
    f3 r_;
    if (dpl2 > 1e-12f) { dp = f_scl(dp, 1.0f / sqrtf(dpl2)); r_ = f_cross(dp, dd); }
    else r_ = E1(a);
    f3 g1 = F3(c * dd.x - s * r_.x, c * dd.y - s * r_.y, c * dd.z - s * r_.z);
    f3 g2 = F3(c * dd.x + s * r_.x, c * dd.y + s * r_.y, c * dd.z + s * r_.z);
    f3 F1 = F3(R * ((-s) * dd.x - c * r_.x), R * ((-s) * dd.y - c * r_.y), R * ((-s) * dd.z - c * r_.z));
    f3 F2 = F3(R * ((-s) * dd.x + c * r_.x), R * ((-s) * dd.y + c * r_.y), R * ((-s) * dd.z + c * r_.z));
    float k1 = f_dot(n, f_sub(p, F1)) / f_dot(n, g1);
    float k2 = f_dot(n, f_sub(p, F2)) / f_dot(n, g2);
    f3 E1v = f_add(F1, f_scl(g1, k1)), E2v = f_add(F2, f_scl(g2, k2));
    *o = f_scl(f_add(E1v, E2v), 0.5f);
    *av = f_scl(f_sub(E1v, E2v), 0.5f);
    float ad = f_dot(*av, dd), aa = f_dot(*av, *av);
    float arg = 1.0f - (ad * ad) / ((c * c) * aa);
    if (arg < 0.0f) arg = 0.0f;
    float lam = sqrtf(arg);
    *bv = f_scl(f_cross(*av, n), lam);
    if (!(f_dot(*bv, *bv) > 1e-12f * aa)) return false;
    return true;
  }

  // end-section (tangency) circle of strut b, parametrised by its strut frame
  __device__ void circle(int b, f3 *o, f3 *av, f3 *bv) const {
    float rs = R * w.s[b], rr = R * w.c[b];
    *o = f_scl(U(b), rs);
    *av = f_scl(E2(b), rr);
    *bv = f_scl(E1(b), rr);
  }
};

__device__ __forceinline__ float conic_t(f3 o, f3 av, f3 bv, f3 P, float *us, float *uc) {
  f3 Q = f_sub(P, o);
  float st = f_dot(Q, av) / f_dot(av, av);
  float ct = f_dot(Q, bv) / f_dot(bv, bv);
  float il = 1.0f / sqrtf(st * st + ct * ct);
  *us = st * il;
  *uc = ct * il;
  return atan2p(st, ct);
}


// Side k >= 1 of a node centred at `on` (.w = R) whose incident strut reaches `pf` (.w = far
// radius); endbit = the node is the strut's i1 end.  Fills the side arrays of ws (w4, wp,
// direction, cone sine/cosine, length, SHORT limit, strut frame).  Returns false for a
// degenerate strut (LMM_NODE_STRUT).  Oracle: build_sides32 / strut_frame32.
template <class WS>
__device__ __forceinline__ bool setup_side(WS &ws, int k, float4 on, float4 pf, int endbit) {
  const float R = on.w;
  f3 po = F3(on.x, on.y, on.z), pfar = F3(pf.x, pf.y, pf.z);
  f3 D = f_sub(pfar, po);
  float Ln = sqrtf(f_dot(D, D));
  if (!(Ln > 0.0f)) return false;
  f3 u = f_div(D, Ln);
  float s = (R - pf.w) / Ln;
  if (!(fabsf(s) < 0.9f)) return false;
  float c = sqrtf(1.0f - s * s);
  f3 wv = f_div(u, c);
  const float ek = (R * s) / c;
  ws.w4[k] = make_float4(wv.x, wv.y, wv.z, ek);
  ws.wp[k][0] = make_float4(wv.x, wv.x, wv.y, wv.y);
  ws.wp[k][1] = make_float4(wv.z, wv.z, -ek, -ek);
  ws.ux[k] = u.x; ws.uy[k] = u.y; ws.uz[k] = u.z;
  ws.s[k] = s; ws.c[k] = c; ws.L[k] = Ln;
  ws.lim[k] = 0.45f * (Ln * c);
  ws.sign[k] = endbit ? -1 : 1;
  // strut frame from p[i1] - p[i0]
  f3 Da = endbit ? f_sub(po, pfar) : f_sub(pfar, po);
  f3 as = f_nrm(Da);
  float ax = fabsf(as.x), ay = fabsf(as.y), az = fabsf(as.z);
  f3 ref = (ax <= ay && ax <= az) ? F3(1.0f, 0.0f, 0.0f) : (ay <= az ? F3(0.0f, 1.0f, 0.0f) : F3(0.0f, 0.0f, 1.0f));
  f3 e1 = f_nrm(f_cross(as, ref));
  f3 e2 = f_cross(as, e1);
  ws.asx[k] = as.x; ws.asy[k] = as.y; ws.asz[k] = as.z;
  ws.e1x[k] = e1.x; ws.e1y[k] = e1.y; ws.e1z[k] = e1.z;
  ws.e2x[k] = e2.x; ws.e2y[k] = e2.y; ws.e2z[k] = e2.z;
  return true;
}

}  // namespace mm
