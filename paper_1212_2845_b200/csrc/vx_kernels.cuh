// vx_kernels.cuh -- sm_100a kernels of the voxel stepper (arXiv:1212.2845).
//
//   k_clock      per-step scalars: t_n, T_n - T_r, motion budget
//   k_dt         K2: stable timestep max-reduction over bonds (Eq. 31-32)
//   k_bonds      K3: per-bond loads (Eq. 13-24, 33-35, 39-40)
//   k_integrate  K4: fixed-order gather (Eq. 25-26), gravity, ground damping,
//                contacts, floor + friction, integration (Eq. 27-30)
//   k_surf_pack  surface table: each slab's surface-voxel state S_n
//   k_broadphase K5: hashed-grid surface-voxel pair list
//   k_contact    self-collision penalty loads on the shortlist
// plus state scatter/gather for the C ABI.  Readings: DESIGN.md §3.
#pragma once
#include "vx_common.cuh"

#include <cooperative_groups.h>
#include <type_traits>

namespace vx {
namespace cg = cooperative_groups;

// Device-resident per-lattice scalars (one allocation).
struct Clock {
  double dT;                    // T_n - T_ref of the step in flight
  long long step;               // index n of the step in flight
  long long next;               // step counter (steps started)
  double budget;                // accumulated max|V| dt since the last rebuild
  unsigned long long vmax_bits; // max |V| of the last update (R bits)
  int rebuild;                  // broadphase runs this step
  int force_rebuild;            // set by set_state / set_environment
  unsigned long long err;       // min over ((step << 32) | box id) of diverged voxels
  unsigned long long fault;     // first step with a non-positive thermal rest length (~0: none)
  int overflow;                 // contact pair list capacity exceeded
  long long npairs;             // pairs a<b in the shortlist
  long long rebuilds;
  unsigned long long w2_bond_bits, w2_vox_bits;  // K2 output (double bits)
};

template <class R> struct Dev {
  using R4 = typename VT<R>::R4;
  using R2 = typename VT<R>::R2;
  R4* pos;
  R4* quat;
  R4* mom;
  R2* ang;
  R4* recA;   // [3][nloc]
  R4* recB;   // [3][nloc]
  R* recC;    // [3][nloc]
  const R4* fext;
  R4* cf;     // contact force per voxel (collision only)
  const int* sidx;   // global surface index of an owned surface voxel, else -1 (collision)
  R4* ss;            // surface table (collision): ss[2s] = pos, ss[2s+1] = mom of S_n
  const MatC<R>* mat;
  const PairC<R>* pair;
  Clock* clk;
  int nmat;
  uint32_t nloc, sx, ny, nz;
  int xl0;            // global x of local plane 0
  R l, half_l, dt;
  double l_d;         // l in fp64: rest sites D0 = origin + l (ijk + 1/2) are formed
                      // in fp64 so the fp32 rounding of l never strains the lattice
  double zbase_d;     // origin_z - floor_z
  int floor_on, ground;
  uint32_t bz;        // layers per z-stacked batched scene (0: none): each scene's floor
                      // sits under its own lowest layer
};

// ------------------------------------------------------------------ clock
struct ClockArgs {
  Clock* clk;
  double dt, T_amp, T_freq, T_phase;
  double half_horizon;   // rebuild when budget >= horizon / 2
  double alpha_lo, alpha_hi;   // extremes of alpha_mean over the lattice's bond pairs
  int collide, precision;
};

__device__ __forceinline__ void clock_tick(const ClockArgs& a) {
  Clock* c = a.clk;
  const long long n = c->next;
  const double t = (double)n * a.dt;
  const double PI = 3.14159265358979323846;
  const double dT = a.T_amp * sin(2 * PI * a.T_freq * t + a.T_phase);
  c->dT = dT;
  // Eq. 40: a rest length l (1 + alpha_mean dT) <= 0 on any bond is a fault
  if (!(1.0 + fmin(a.alpha_lo * dT, a.alpha_hi * dT) > 0.0) && (unsigned long long)n < c->fault)
    c->fault = (unsigned long long)n;
  c->step = n;
  c->next = n + 1;
  if (a.collide) {
    double vmax = a.precision == 32 ? (double)__uint_as_float((unsigned)c->vmax_bits)
                                    : __longlong_as_double((long long)c->vmax_bits);
    c->vmax_bits = 0;
    double b = c->budget + vmax * a.dt;
    if (c->force_rebuild || b >= a.half_horizon) {
      c->rebuild = 1;
      c->force_rebuild = 0;
      b = 0;
    } else {
      c->rebuild = 0;
    }
    c->budget = b;
  }
}
__global__ void k_clock(ClockArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  clock_tick(a);
}

// ------------------------------------------------------------------ K2 dt
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// w2 of a bond = a1 / m_min (pair table, fp64); w2 of a voxel = E l / m.
template <class R>
__global__ void __launch_bounds__(256) k_dt(const typename VT<R>::R4* pos, uint32_t beg,
                                            uint32_t end, uint32_t sx, uint32_t nz,
                                            const double* pair_w2, const double* mat_w2,
                                            int nmat, Clock* clk) {
  __shared__ double sb[8], sv[8];
  const uint32_t id = beg + blockIdx.x * blockDim.x + threadIdx.x;
  double wb = 0, wv = 0;
  if (id < end) {
    uint32_t m = meta_of(pos[id].w);
    if (m & M_FILLED) {
      int ma = m & M_MAT;
      wv = mat_w2[ma];
      const uint32_t strides[3] = {sx, nz, 1u};
#pragma unroll
      for (int ax = 0; ax < 3; ++ax)
        if (m & nb_bit(2 * ax + 1)) {
          int mb = meta_of(pos[id + strides[ax]].w) & M_MAT;
          wb = fmax(wb, pair_w2[ma * nmat + mb]);
        }
    }
  }
  wb = warp_max(wb);
  wv = warp_max(wv);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sb[warp] = wb; sv[warp] = wv; }
  __syncthreads();
  if (warp == 0) {
    wb = lane < (int)(blockDim.x >> 5) ? sb[lane] : 0.0;
    wv = lane < (int)(blockDim.x >> 5) ? sv[lane] : 0.0;
    wb = warp_max(wb);
    wv = warp_max(wv);
    if (lane == 0) {   // positive doubles order like their bit patterns
      atomicMax(&clk->w2_bond_bits, (unsigned long long)__double_as_longlong(wb));
      atomicMax(&clk->w2_vox_bits, (unsigned long long)__double_as_longlong(wv));
    }
  }
}

// ------------------------------------------------------------------ K3 bonds
// Scale k with theta = k v for the unit quaternion (w >= 0, |v| = s):
// k = 2 atan2(s, w) / s (reading R7).  Bond rotations are small (the beam
// model's own range), so for s below a threshold the identity
// 2 atan2(s, w) = 2 asin(s) (w = sqrt(1 - s^2)) is used through its series
// 2 asin(s)/s = 2 (1 + s^2/6 + 3 s^4/40 + 5 s^6/112 + 35 s^8/1152), truncated
// where the next term is below the type's rounding: no division, no atan2.
template <class R> struct SeriesCut;
template <> struct SeriesCut<float> { static constexpr float s2 = 0.125f * 0.125f; };
template <> struct SeriesCut<double> { static constexpr double s2 = 0.002 * 0.002; };
template <class R> __device__ __forceinline__ R rotvec_scale(R w, R x, R y, R z) {
  const R s2 = xdot3(x, x, y, y, z, z);
  if (s2 < SeriesCut<R>::s2) {
    return xfma(s2, xfma(s2, xfma(s2, xfma(s2, R(35) / R(576), R(5) / R(56)), R(3) / R(20)),
                         R(1) / R(3)), R(2));
  }
  const R s = vx_sqrt(s2);
  return xmul(R(2), vx_atan2(s, w)) / s;
}

// Voxel a (negative side, R4) and b = a + e_AX.  Loads in the frame of a
// (P:189), Eq. 13-24 sign-fixed and negated (R1, R3), back to world,
// plus local damping (Eq. 33-35, R10, R11).  Shared by K3 and the fused step.
template <class R> struct VS {   // one voxel's state as loaded
  typename VT<R>::R4 p, q, mo;   // (u, meta), quaternion (x,y,z,w), (P, phi.z)
  typename VT<R>::R2 an;         // (phi.x, phi.y)
};
template <class R>
__device__ __forceinline__ VS<R> ld_vs(const typename VT<R>::R4* __restrict__ pos,
                                       const typename VT<R>::R4* __restrict__ quat,
                                       const typename VT<R>::R4* __restrict__ mom,
                                       const typename VT<R>::R2* __restrict__ ang, uint32_t i) {
  VS<R> s;
  s.p = pos[i];
  s.q = quat[i];
  s.mo = mom[i];
  s.an = ang[i];
  return s;
}

// A voxel's state by local id (bounds-checked in the checked build).
template <class R> __device__ __forceinline__ VS<R> ldv(const Dev<R>& d, uint32_t i) {
  VX_CHK(i < d.nloc, 1);
  return ld_vs<R>(d.pos, d.quat, d.mom, d.ang, i);
}

template <int AX, class R>
__device__ __forceinline__ void bond_eval(const Dev<R>& d, const Rot<R>& Ra,
                                          const typename VT<R>::R4& qa, V3<R> ua, V3<R> Va,
                                          V3<R> wa, int mat_a, const VS<R>& b, R dT, V3<R>& Fa,
                                          V3<R>& Ma, V3<R>& Mbw) {
  using R4 = typename VT<R>::R4;
  const R4& pb = b.p;
  const R4& qb = b.q;
  const int mat_b = meta_of(pb.w) & M_MAT;
  VX_CHK(mat_a < d.nmat && mat_b < d.nmat, 4);
  const PairC<R> c = d.pair[mat_a * d.nmat + mat_b];
  const R l = d.l;

  // relative position in a's frame, cancellation-free:
  //   R^T r - l e = l (R^T e - e) + R^T (u_b - u_a)
  const V3<R> du = xsub3(mk(pb.x, pb.y, pb.z), ua);
  V3<R> t;  // R^T e_AX - e_AX = row AX of (R - I)
  if constexpr (AX == 0) t = mk(Ra.dd[0], Ra.m[0][1], Ra.m[0][2]);
  else if constexpr (AX == 1) t = mk(Ra.m[1][0], Ra.dd[1], Ra.m[1][2]);
  else t = mk(Ra.m[2][0], Ra.m[2][1], Ra.dd[2]);
  const V3<R> dv = to_bond<AX>(xfma3(l, t, mulT(Ra, du)));

  // relative rotation theta = rotvec(q_a* q_b), w >= 0 (R6, R7); each
  // component summed a_w b + a_x b + a_y b + a_z b, left to right
  const R qw = xfma(qa.z, qb.z, xfma(qa.y, qb.y, xfma(qa.x, qb.x, xmul(qa.w, qb.w))));
  const R qx = xfma(qa.z, qb.y, xfma(-qa.y, qb.z, xfma(-qa.x, qb.w, xmul(qa.w, qb.x))));
  const R qy = xfma(-qa.z, qb.x, xfma(-qa.y, qb.w, xfma(qa.x, qb.z, xmul(qa.w, qb.y))));
  const R qz = xfma(-qa.z, qb.w, xfma(qa.y, qb.x, xfma(-qa.x, qb.y, xmul(qa.w, qb.z))));
  // w < 0: theta of -q_rel (the same rotation); the sign folds into the scale
  const R kth = (qw < R(0) ? R(-1) : R(1)) * rotvec_scale(fabs(qw), qx, qy, qz);
  const V3<R> th = to_bond<AX>(xscale3(kth, mk(qx, qy, qz)));

  // Eq. 40: X2 = d_x - L_T with L_T = l (1 + alpha_mean dT)
  const R X2 = xsub(dv.x, xmul(xmul(l, c.alpha_mean), dT));
  const R Y2 = dv.y, Z2 = dv.z;
  const R b3x2 = R(2) * c.b3;
  const V3<R> fa = mk(xmul(c.a1, X2), xfma(-c.b2, th.z, xmul(c.b1, Y2)),
                      xfma(c.b2, th.y, xmul(c.b1, Z2)));
  const V3<R> ma = mk(xmul(c.a2, th.x), xfma(-c.b3, th.y, xmul(-c.b2, Z2)),
                      xfma(-c.b3, th.z, xmul(c.b2, Y2)));
  const V3<R> mbl = mk(xmul(-c.a2, th.x), xfma(-b3x2, th.y, xmul(-c.b2, Z2)),
                       xfma(-b3x2, th.z, xmul(c.b2, Y2)));
  Fa = mul(Ra, to_world<AX>(fa));
  Ma = mul(Ra, to_world<AX>(ma));
  Mbw = mul(Ra, to_world<AX>(mbl));

  // Eq. 33-35 in the world frame.  With the averages written out,
  //   V_r = (V_b - V_avg) + (r/2) x w_avg = (V_b - V_a)/2 + (r x (w_a + w_b))/4
  //   w_r = w_b - w_avg = (w_b - w_a)/2
  // and c_t/2, c_t/4, c_r/2 come from the pair table (exact power-of-2 scalings).
  const V3<R> Vb = xscale3(c.inv_m_b, mk(b.mo.x, b.mo.y, b.mo.z));
  const V3<R> wb = xscale3(c.inv_I_b, mk(b.an.x, b.an.y, b.mo.w));
  V3<R> r = du;
  if constexpr (AX == 0) r.x = xadd(r.x, l);
  else if constexpr (AX == 1) r.y = xadd(r.y, l);
  else r.z = xadd(r.z, l);
  const V3<R> dV = xsub3(Vb, Va);
  const V3<R> rw = xcross(r, xadd3(wa, wb));
  const V3<R> dw = xsub3(wb, wa);
  Fa = xfma3(c.ct4, rw, xfma3(c.ct2, dV, Fa));
  Ma = xfma3(c.cr2, dw, Ma);
  Mbw = xfma3(-c.cr2, dw, Mbw);
}

// fp32 bond: the same operations in the same order as the generic bond_eval,
// with 2-vector work on the FP32x2 path (vx_common.cuh): the relative
// quaternion as two pair products (qx, qy), (qz, qw); rotations back to the
// world frame by column pairs; velocities and the damping sums paired.
// Pairs used: (u, P).xy from the float4 loads, (phi_x, phi_y) from the
// float2 load, (x, y) / (z, w) of each quaternion.
template <int AX>
__device__ __forceinline__ void bond_eval(const Dev<float>& d, const RotP& Ra, const float4& qa,
                                          V3<float> ua, V3<float> Va, V3<float> wa, int mat_a,
                                          const VS<float>& b, float dT, V3<float>& Fa,
                                          V3<float>& Ma, V3<float>& Mbw) {
  const float4& pb = b.p;
  const float4& qb = b.q;
  const int mat_b = meta_of(pb.w) & M_MAT;
  VX_CHK(mat_a < d.nmat && mat_b < d.nmat, 4);
  const PairC<float> c = d.pair[mat_a * d.nmat + mat_b];
  const float l = d.l;

  const f2_t duxy = sub2(f2pk(pb.x, pb.y), f2pk(ua.x, ua.y));
  const V3<float> du = mk(f2lo(duxy), f2hi(duxy), xsub(pb.z, ua.z));
  V3<float> t;  // R^T e_AX - e_AX = row AX of (R - I)
  if constexpr (AX == 0) t = mk(Ra.dd0, f2lo(Ra.c1), f2lo(Ra.c2));
  else if constexpr (AX == 1) t = mk(f2hi(Ra.c0), Ra.dd1, f2hi(Ra.c2));
  else t = mk(Ra.m20, Ra.m21, Ra.dd2);
  const V3<float> dv = to_bond<AX>(xfma3(l, t, mulT(Ra, du)));

  // q_rel = q_a* q_b as two pair products, q_a's components broadcast (the
  // scalar operand of FFMA2 / FMUL2) against signed, swapped pairs of q_b:
  //   (qx, qy) = aw (bx, by) + ax (-bw, bz) - ay (bz, bw) + az (by, -bx)
  //   (qz, qw) = aw (bz, bw) + ax (-by, bx) + ay (bx, by) + az (-bw, bz)
  // (per lane the same fma chain as the scalar formula: ax (-bw) = (-ax) bw
  // exactly; signs on q_a's side made the compiler materialise broadcast pairs)
  const f2_t B1 = f2pk(qb.x, qb.y), B2 = f2pk(qb.z, qb.w);
  const f2_t Wn = f2pk(-qb.w, qb.z), Yn = f2pk(qb.y, -qb.x), Yp = f2pk(-qb.y, qb.x);
  const f2_t qxy = fma2(bc2(qa.z), Yn, fma2(bc2(-qa.y), B2, fma2(bc2(qa.x), Wn, mul2(bc2(qa.w), B1))));
  const f2_t qzw = fma2(bc2(qa.z), Wn, fma2(bc2(qa.y), B1, fma2(bc2(qa.x), Yp, mul2(bc2(qa.w), B2))));
  const float qx = f2lo(qxy), qy = f2hi(qxy), qz = f2lo(qzw), qw = f2hi(qzw);
  const float kth = (qw < 0.f ? -1.f : 1.f) * rotvec_scale(fabsf(qw), qx, qy, qz);
  const f2_t thxy = mul2(bc2(kth), qxy);
  const V3<float> th = to_bond<AX>(mk(f2lo(thxy), f2hi(thxy), xmul(kth, qz)));

  const float X2 = xsub(dv.x, xmul(xmul(l, c.alpha_mean), dT));
  const float Y2 = dv.y, Z2 = dv.z;
  const float b3x2 = 2.f * c.b3;
  // the generic formulas, paired (same roundings, lane by lane):
  //   (fa.x, ma.x) = (a1, a2) (X2, th.x);  mbl.x = -ma.x (exact)
  //   (fa.y, fa.z) = (-b2, b2) (th.z, th.y) + b1 (Y2, Z2)
  //   (ma.y, ma.z) = -b3 (th.y, th.z) + (-b2, b2) (Z2, Y2)
  //   (mbl.y, mbl.z) = -2 b3 (th.y, th.z) + (-b2, b2) (Z2, Y2)
  const f2_t nbb = f2pk(c.nb2, c.b2);
  const f2_t xa = mul2(f2pk(c.a1, c.a2), f2pk(X2, th.x));
  const f2_t fyz = fma2(nbb, f2pk(th.z, th.y), mul2(bc2(c.b1), f2pk(Y2, Z2)));
  const f2_t pzy = mul2(nbb, f2pk(Z2, Y2));
  const f2_t thyz = f2pk(th.y, th.z);
  const f2_t myz = fma2(bc2(-c.b3), thyz, pzy);
  const f2_t byz = fma2(bc2(-b3x2), thyz, pzy);
  const V3<float> fa = mk(f2lo(xa), f2lo(fyz), f2hi(fyz));
  const V3<float> ma = mk(f2hi(xa), f2lo(myz), f2hi(myz));
  const V3<float> mbl = mk(-f2hi(xa), f2lo(byz), f2hi(byz));
  Fa = mul(Ra, to_world<AX>(fa));
  Ma = mul(Ra, to_world<AX>(ma));
  Mbw = mul(Ra, to_world<AX>(mbl));

  // Eq. 33-35 (see the generic bond_eval)
  const f2_t Vbxy = mul2(bc2(c.inv_m_b), f2pk(b.mo.x, b.mo.y));
  const float Vbz = xmul(c.inv_m_b, b.mo.z);
  const f2_t wbxy = mul2(bc2(c.inv_I_b), f2pk(b.an.x, b.an.y));
  const float wbz = xmul(c.inv_I_b, b.mo.w);
  V3<float> r = du;
  if constexpr (AX == 0) r.x = xadd(r.x, l);
  else if constexpr (AX == 1) r.y = xadd(r.y, l);
  else r.z = xadd(r.z, l);
  const f2_t waxy = f2pk(wa.x, wa.y);
  const f2_t dVxy = sub2(Vbxy, f2pk(Va.x, Va.y));
  const float dVz = xsub(Vbz, Va.z);
  const f2_t sxy = add2(waxy, wbxy);
  const V3<float> rw = xcross(r, mk(f2lo(sxy), f2hi(sxy), xadd(wa.z, wbz)));
  const f2_t dwxy = sub2(wbxy, waxy);
  const float dwz = xsub(wbz, wa.z);
  const f2_t Fxy = fma2(bc2(c.ct4), f2pk(rw.x, rw.y), fma2(bc2(c.ct2), dVxy, f2pk(Fa.x, Fa.y)));
  Fa = mk(f2lo(Fxy), f2hi(Fxy), fmaf(c.ct4, rw.z, fmaf(c.ct2, dVz, Fa.z)));
  const f2_t Mxy = fma2(bc2(c.cr2), dwxy, f2pk(Ma.x, Ma.y));
  Ma = mk(f2lo(Mxy), f2hi(Mxy), fmaf(c.cr2, dwz, Ma.z));
  const f2_t Bxy = fma2(bc2(-c.cr2), dwxy, f2pk(Mbw.x, Mbw.y));
  Mbw = mk(f2lo(Bxy), f2hi(Bxy), fmaf(-c.cr2, dwz, Mbw.z));
}

// The parts of voxel a that every bond of a shares.
template <class R> struct RotOf { using T = Rot<R>; };
template <> struct RotOf<float> { using T = RotP; };
template <class R> struct AFrame {
  typename RotOf<R>::T Ra;
  V3<R> ua, Va, wa;
  int mat;
};
template <class R> __device__ __forceinline__ AFrame<R> a_frame(const Dev<R>& d, const VS<R>& a) {
  AFrame<R> f;
  const uint32_t meta = meta_of(a.p.w);
  f.mat = meta & M_MAT;
  const MatC<R>& M = d.mat[f.mat];
  f.ua = mk(a.p.x, a.p.y, a.p.z);
  if constexpr (sizeof(R) == 4) {
    f.Ra = rotation_p(a.q.x, a.q.y, a.q.z, a.q.w);
    const f2_t vxy = mul2(bc2(M.inv_m), f2pk(a.mo.x, a.mo.y));
    const f2_t wxy = mul2(bc2(M.inv_I), f2pk(a.an.x, a.an.y));
    f.Va = mk(f2lo(vxy), f2hi(vxy), xmul(M.inv_m, a.mo.z));
    f.wa = mk(f2lo(wxy), f2hi(wxy), xmul(M.inv_I, a.mo.w));
  } else {
    f.Ra = rotation(a.q.w, a.q.x, a.q.y, a.q.z);
    f.Va = xscale3(M.inv_m, mk(a.mo.x, a.mo.y, a.mo.z));
    f.wa = xscale3(M.inv_I, mk(a.an.x, a.an.y, a.mo.w));
  }
  return f;
}

template <int AX, class R>
__device__ __forceinline__ void bond_one(const Dev<R>& d, uint32_t ia, uint32_t ib,
                                         const AFrame<R>& f, const typename VT<R>::R4& qa, R dT) {
  using R4 = typename VT<R>::R4;
  const VS<R> b = ldv(d, ib);
  V3<R> Fa, Ma, Mbw;
  bond_eval<AX>(d, f.Ra, qa, f.ua, f.Va, f.wa, f.mat, b, dT, Fa, Ma, Mbw);
  const size_t o = (size_t)AX * d.nloc + ia;
  d.recA[o] = R4{Fa.x, Fa.y, Fa.z, Ma.x};
  d.recB[o] = R4{Ma.y, Ma.z, Mbw.x, Mbw.y};
  d.recC[o] = Mbw.z;
}

template <class R>
__global__ void __launch_bounds__(256, sizeof(R) == 4 ? 4 : 2) k_bonds(Dev<R> d, uint32_t beg, uint32_t end) {
  const uint32_t id = beg + blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= end) return;
  const typename VT<R>::R4 pa = d.pos[id];
  const uint32_t meta = meta_of(pa.w);
  const uint32_t want = meta & (nb_bit(1) | nb_bit(3) | nb_bit(5));
  if (!want) return;
  VS<R> a;
  a.p = pa;
  a.q = d.quat[id];
  a.mo = d.mom[id];
  a.an = d.ang[id];
  const AFrame<R> f = a_frame(d, a);
  const R dT = (R)d.clk->dT;
  if (want & nb_bit(1)) bond_one<0>(d, id, id + d.sx, f, a.q, dT);
  if (want & nb_bit(3)) bond_one<1>(d, id, id + d.nz, f, a.q, dT);
  if (want & nb_bit(5)) bond_one<2>(d, id, id + 1, f, a.q, dT);
}

// ------------------------------------------------------------------ K4 integrate
// Rotation increment below IncCut's squared angle uses the series of cos(a/2)
// and sin(a/2)/a through a^6 (next term < 1e-17 relative at the cut).

// Stores of the new state are never re-read by the same kernel: evict-first.
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float2* p, float2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double4* p, double4 v) {
  double2* q = reinterpret_cast<double2*>(p);
  __stcs(q, make_double2(v.x, v.y));
  __stcs(q + 1, make_double2(v.z, v.w));
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }

// Eq. 27-30 and the store of S_{n+1}: P += F dt, D += (P/m) dt, phi += M dt,
// q <- normalize(quat(th) (x) q), quat(th) = (cos(a/2), sin(a/2) th/a),
// th = (phi/I) dt, a = |th|; returns |V| for the motion budget.
template <class R> struct IncCut;
template <> struct IncCut<float> { static constexpr float a2 = 0.05f * 0.05f; };
template <> struct IncCut<double> { static constexpr double a2 = 0.01 * 0.01; };
// cos(a/2) and sin(a/2)/a of the per-step rotation increment
template <class R> __device__ __forceinline__ void inc_coeffs(R a2, R& dw, R& ks) {
  if (a2 < IncCut<R>::a2) {   // per-step angles are tiny: Taylor series, no sincos
    dw = R(1) - a2 * (R(1) / R(8) - a2 * (R(1) / R(384) - a2 * (R(1) / R(46080))));
    ks = R(0.5) - a2 * (R(1) / R(48) - a2 * (R(1) / R(3840) - a2 * (R(1) / R(645120))));
  } else {
    const R a = vx_sqrt(a2);
    R sh;
    vx_sincos(R(0.5) * a, &sh, &dw);
    ks = sh / a;
  }
}
template <class R> __device__ __forceinline__ void flag_nonfinite(const Dev<R>& d, uint32_t id, R z,
                                                                  const uint32_t* ext_of_local) {
  if (!(z == R(0))) {
    const unsigned long long code =
        ((unsigned long long)d.clk->step << 32) | (unsigned long long)ext_of_local[id];
    atomicMin(&d.clk->err, code);
  }
}
// A surface voxel's new state also goes to the surface table, so the next
// step's contact front reads it without a separate pack (k_surf_pack only
// initialises the table after a state change).
template <class R>
__device__ __forceinline__ void surface_entry(const Dev<R>& d, uint32_t id, uint32_t nmeta,
                                              const typename VT<R>::R4& npos,
                                              const typename VT<R>::R4& nmom) {
  if (!(nmeta & M_SURF)) return;
  const int s = d.sidx[id];
  if (s < 0) return;
  d.ss[2 * s] = npos;
  d.ss[2 * s + 1] = nmom;
}
template <class R, bool COLLIDE>
__device__ __forceinline__ R integrate_store(const Dev<R>& d, uint32_t id, const VS<R>& s,
                                             uint32_t nmeta, const MatC<R>& mc, V3<R> F, V3<R> M,
                                             bool zero_lat, typename VT<R>::R4* __restrict__ opos,
                                             typename VT<R>::R4* __restrict__ oquat,
                                             typename VT<R>::R4* __restrict__ omom,
                                             typename VT<R>::R2* __restrict__ oang,
                                             const uint32_t* __restrict__ ext_of_local) {
  using R4 = typename VT<R>::R4;
  using R2 = typename VT<R>::R2;
  const R4& p = s.p;
  const R4& mo = s.mo;
  V3<R> P = mk(mo.x, mo.y, mo.z) + d.dt * F;
  if (zero_lat) { P.x = R(0); P.y = R(0); }
  const V3<R> u = mk(p.x, p.y, p.z) + mc.dt_m * P;
  const V3<R> phi = mk(s.an.x, s.an.y, mo.w) + d.dt * M;
  const V3<R> th = mc.dt_I * phi;
  R dw, ks;
  inc_coeffs(dot(th, th), dw, ks);
  const R dx = ks * th.x, dy = ks * th.y, dz = ks * th.z;
  const R4& q = s.q;
  R qw = dw * q.w - dx * q.x - dy * q.y - dz * q.z;
  R qx = dw * q.x + dx * q.w + dy * q.z - dz * q.y;
  R qy = dw * q.y - dx * q.z + dy * q.w + dz * q.x;
  R qz = dw * q.z + dx * q.y - dy * q.x + dz * q.w;
  const R qi = vx_rnorm(qw * qw + qx * qx + qy * qy + qz * qz);
  qw = qw * qi; qx = qx * qi; qy = qy * qi; qz = qz * qi;
  const R4 npos{u.x, u.y, u.z, meta_as(R(0), nmeta)}, nmom{P.x, P.y, P.z, phi.z};
  st_stream(opos + id, npos);
  st_stream(oquat + id, R4{qx, qy, qz, qw});
  st_stream(omom + id, nmom);
  st_stream(oang + id, R2{phi.x, phi.y});
  if constexpr (COLLIDE) surface_entry(d, id, nmeta, npos, nmom);
  // any NaN/Inf among the 13 values: x * 0 is NaN exactly for non-finite x
  const R z0 = (u.x + u.y + u.z + qw + qx + qy + qz) * R(0);
  const R z1 = (P.x + P.y + P.z + phi.x + phi.y + phi.z) * R(0);
  flag_nonfinite(d, id, z0 + z1, ext_of_local);
  return COLLIDE ? vx_sqrt(dot(P, P)) * mc.inv_m : R(0);
}
// fp32: the same steps with (x, y) of P, D, phi, th and the two halves
// (x, y), (z, w) of the quaternion product on the FP32x2 path.
//   (qx', qy') = dw (qx, qy) - dx (-qw, qz) + dy (qz, qw) + dz (-qy, qx)
//   (qz', qw') = dw (qz, qw) - dx (-qy, qx) - dy (qx, qy) - dz (-qw, qz)
template <bool COLLIDE>
__device__ __forceinline__ float integrate_store_f32(const Dev<float>& d, uint32_t id, const VS<float>& s,
                                                 uint32_t nmeta, const MatC<float>& mc, V3<float> F,
                                                 V3<float> M, bool zero_lat, float4* __restrict__ opos,
                                                 float4* __restrict__ oquat, float4* __restrict__ omom,
                                                 float2* __restrict__ oang,
                                                 const uint32_t* __restrict__ ext_of_local) {
  const float4& p = s.p;
  const float4& mo = s.mo;
  f2_t Pxy = fma2(bc2(d.dt), f2pk(F.x, F.y), f2pk(mo.x, mo.y));
  const float Pz = fmaf(d.dt, F.z, mo.z);
  if (zero_lat) Pxy = zero2();
  const f2_t uxy = fma2(bc2(mc.dt_m), Pxy, f2pk(p.x, p.y));
  const float uz = fmaf(mc.dt_m, Pz, p.z);
  const f2_t phxy = fma2(bc2(d.dt), f2pk(M.x, M.y), f2pk(s.an.x, s.an.y));
  const float phz = fmaf(d.dt, M.z, mo.w);
  const f2_t thxy = mul2(bc2(mc.dt_I), phxy);
  const float thx = f2lo(thxy), thy = f2hi(thxy), thz = mc.dt_I * phz;
  float dw, ks;
  inc_coeffs(thx * thx + thy * thy + thz * thz, dw, ks);
  const f2_t dxy = mul2(bc2(ks), thxy);
  const float dx = f2lo(dxy), dy = f2hi(dxy), dz = ks * thz;
  const float4& q = s.q;
  const f2_t Q1 = f2pk(q.x, q.y), Q2 = f2pk(q.z, q.w);
  const f2_t nQ1 = f2pk(-q.y, q.x), nQ2 = f2pk(-q.w, q.z);
  f2_t q1 = fma2(bc2(dz), nQ1, fma2(bc2(dy), Q2, fma2(bc2(-dx), nQ2, mul2(bc2(dw), Q1))));
  f2_t q2 = fma2(bc2(-dz), nQ2, fma2(bc2(-dy), Q1, fma2(bc2(-dx), nQ1, mul2(bc2(dw), Q2))));
  const f2_t nn = fma2(q1, q1, mul2(q2, q2));
  const float qi = vx_rnorm(f2lo(nn) + f2hi(nn));
  q1 = mul2(bc2(qi), q1);
  q2 = mul2(bc2(qi), q2);
  const float4 npos{f2lo(uxy), f2hi(uxy), uz, meta_as(0.f, nmeta)};
  const float4 nmom{f2lo(Pxy), f2hi(Pxy), Pz, phz};
  st_stream(opos + id, npos);
  st_stream(oquat + id, float4{f2lo(q1), f2hi(q1), f2lo(q2), f2hi(q2)});
  st_stream(omom + id, nmom);
  st_stream(oang + id, float2{f2lo(phxy), f2hi(phxy)});
  if constexpr (COLLIDE) surface_entry(d, id, nmeta, npos, nmom);
  // any NaN/Inf among the 13 values: x * 0 is NaN exactly for non-finite x
  const f2_t sxy = add2(add2(add2(add2(uxy, q1), q2), Pxy), phxy);
  flag_nonfinite(d, id, (f2lo(sxy) + f2hi(sxy) + uz + Pz + phz) * 0.f, ext_of_local);
  if constexpr (COLLIDE) {
    const f2_t pp = mul2(Pxy, Pxy);
    return vx_sqrt(f2lo(pp) + f2hi(pp) + Pz * Pz) * mc.inv_m;
  }
  return 0.f;
}

// Layer of global layer k within its z-stacked batched scene (vx_set_batch_z):
// the floor lies under each scene's own lowest layer.
template <class R> __device__ __forceinline__ uint32_t floor_layer(const Dev<R>& d, uint32_t k) {
  return d.bz ? k % d.bz : k;
}
// Height of the rest site of layer k above the floor, D0_z - z_floor, formed in
// fp64 (Dev::l_d) and rounded to R once; layer k within its scene (floor_layer).
template <class R> __device__ __forceinline__ R floor_base(const Dev<R>& d, uint32_t k) {
  return (R)(d.zbase_d + d.l_d * (double)floor_layer(d, k));
}

// After the slot sums (Eq. 25-26): external force, gravity, ground
// damping (R12), contacts, floor + friction (R14, R15),
// integration (Eq. 27-30); writes the new state of `id` to the out arrays.
// zb: floor_base of the voxel's layer (the fused pass forms it once per thread).
template <class R, bool COLLIDE>
__device__ __forceinline__ R finish_voxel(const Dev<R>& d, uint32_t id, R zb, const VS<R>& s,
                                          uint32_t meta,
                                          V3<R> F, V3<R> M, typename VT<R>::R4* __restrict__ opos,
                                          typename VT<R>::R4* __restrict__ oquat,
                                          typename VT<R>::R4* __restrict__ omom,
                                          typename VT<R>::R2* __restrict__ oang,
                                          const uint32_t* __restrict__ ext_of_local) {
  using R4 = typename VT<R>::R4;
  VX_CHK(id < d.nloc, 7);
  VX_CHK((int)(meta & M_MAT) < d.nmat, 4);
  const MatC<R> mc = d.mat[meta & M_MAT];
  const R4& p = s.p;
  const R4& mo = s.mo;
  if (meta & M_EXT) {
    const R4 fe = d.fext[id];
    F = F + mk(fe.x, fe.y, fe.z);
  }
  F.z = F.z - mc.mg;
  V3<R> V;
  if constexpr (sizeof(R) == 4) {
    const f2_t vxy = mul2(bc2(mc.inv_m), f2pk(mo.x, mo.y));
    V = mk(f2lo(vxy), f2hi(vxy), mc.inv_m * mo.z);
    if (d.ground) {                                   // P:254, R12
      const f2_t wxy = mul2(bc2(mc.inv_I), f2pk(s.an.x, s.an.y));
      const f2_t fxy = fma2(bc2(-mc.cgt), vxy, f2pk(F.x, F.y));
      const f2_t mxy = fma2(bc2(-mc.cgr), wxy, f2pk(M.x, M.y));
      F = mk(f2lo(fxy), f2hi(fxy), fmaf(-mc.cgt, V.z, F.z));
      M = mk(f2lo(mxy), f2hi(mxy), fmaf(-mc.cgr, mc.inv_I * mo.w, M.z));
    }
  } else {
    V = mc.inv_m * mk(mo.x, mo.y, mo.z);
    if (d.ground) {                                   // P:254, R12
      F = F - mc.cgt * V;
      M = M - mc.cgr * (mc.inv_I * mk(s.an.x, s.an.y, mo.w));
    }
  }
  if constexpr (COLLIDE) {
    if (meta & M_SURF) {
      const R4 c = d.cf[id];
      F = F + mk(c.x, c.y, c.z);
    }
  }
  bool latch = (meta & M_LATCH) != 0;
  bool zero_lat = false;
  if (d.floor_on) {                                   // P:260-274, R14, R15
    const R dT = (R)d.clk->dT;
    // penetration r_v - (D_z - z_floor), r_v = (l/2)(1 + alpha dT)
    const R pen = d.half_l * mc.alpha * dT - p.z - zb;
    if (pen > R(0)) {
      R Fn = mc.kf * pen - mc.cfl * V.z;
      if (Fn < R(0)) Fn = R(0);
      F.z = F.z + Fn;
      const R Flx = F.x, Fly = F.y;
      const R Fl = vx_sqrt(Flx * Flx + Fly * Fly);
      const R Vl = vx_sqrt(V.x * V.x + V.y * V.y);
      if (latch) {
        if (Fl <= mc.mu_s * Fn) {                     // Eq. 36 holds
          F.x = R(0); F.y = R(0); zero_lat = true;
        } else {                                      // break away, Eq. 37
          latch = false;
          F.x = Flx - mc.mu_d * Fn * Flx / Fl;
          F.y = Fly - mc.mu_d * Fn * Fly / Fl;
        }
      } else {
        if (Vl <= mc.mu_d * Fn * mc.dt_m) {           // Eq. 38 halt
          F.x = R(0); F.y = R(0); zero_lat = true; latch = true;
        } else {
          F.x = Flx - mc.mu_d * Fn * V.x / Vl;
          F.y = Fly - mc.mu_d * Fn * V.y / Vl;
        }
      }
    } else {
      latch = false;
    }
  }
  const uint32_t nmeta = latch ? (meta | M_LATCH) : (meta & ~M_LATCH);
  if constexpr (sizeof(R) == 4)
    return integrate_store_f32<COLLIDE>(d, id, s, nmeta, mc, F, M, zero_lat, opos, oquat, omom,
                                        oang, ext_of_local);
  else
    return integrate_store<R, COLLIDE>(d, id, s, nmeta, mc, F, M, zero_lat, opos, oquat, omom,
                                       oang, ext_of_local);
}

// Block max of |V| -> motion budget.  All threads of the block call it.
template <class R> __device__ __forceinline__ void budget_max(const Dev<R>& d, R v) {
  __shared__ R sm[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sm[lane] : R(0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0 && v > R(0)) {
      using UB = typename VT<R>::UB;
      atomicMax((UB*)&d.clk->vmax_bits, (UB)rbits(v));
    }
  }
}

template <class R, bool COLLIDE>
__global__ void __launch_bounds__(256) k_integrate(Dev<R> d, uint32_t beg, uint32_t end,
                                                   const uint32_t* __restrict__ ext_of_local) {
  using R4 = typename VT<R>::R4;
  const uint32_t id = beg + blockIdx.x * blockDim.x + threadIdx.x;
  R vmax = R(0);
  if (id < end) {
    const R4 p = d.pos[id];
    const uint32_t meta = meta_of(p.w);
    if ((meta & (M_FILLED | M_FIXED)) == M_FILLED) {
      VS<R> s;
      s.p = p;
      s.mo = d.mom[id];
      s.an = d.ang[id];
      V3<R> F = mk(R(0), R(0), R(0)), M = F;
      const uint32_t strides[3] = {d.sx, d.nz, 1u};
      // Eq. 25-26 in slot order -x,+x,-y,+y,-z,+z: a -axis slot holds the
      // bond (v-e, v) where v is "b" (-F_a, M_b); a +axis slot (F_a, M_a).
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        if (meta & nb_bit(2 * ax)) {
          const size_t o = (size_t)ax * d.nloc + (id - strides[ax]);
          const R4 A = d.recA[o];
          const R4 B = d.recB[o];
          const R C = d.recC[o];
          F = F - mk(A.x, A.y, A.z);
          M = M + mk(B.z, B.w, C);
        }
        if (meta & nb_bit(2 * ax + 1)) {
          const size_t o = (size_t)ax * d.nloc + id;
          const R4 A = d.recA[o];
          const R4 B = d.recB[o];
          F = F + mk(A.x, A.y, A.z);
          M = M + mk(A.w, B.x, B.y);
        }
      }
      s.q = d.quat[id];
      vmax = finish_voxel<R, COLLIDE>(d, id, floor_base(d, id % d.nz), s, meta, F, M, d.pos, d.quat, d.mom, d.ang,
                                      ext_of_local);
    }
  }
  if constexpr (COLLIDE) budget_max(d, vmax);
}

// ------------------------------------------------------------------ fused step (NEXT f1)
// One pass per step: reads S_n (in), writes S_{n+1} (out), bond loads never
// touch HBM.  A block owns rows [j0, j0+TY) of x-planes [i0, i1) over the full
// z range (thread = k, nz <= blockDim.x) and sweeps x.  Per voxel it computes
// its +x, +y, +z bonds exactly as K3 does (bond_eval); the -x slot is its own
// previous-plane +x bond (shared memory), the -y slot its previous row's +y
// bond (registers), the -z slot the +z bond of thread k-1 (shared memory).
// Halo: the +y bond of row j0-1 per plane and the +x bond of plane i0-1 per
// segment are recomputed.  The slot sums and finish_voxel are K4's, in K4's
// order, so the update is the two-kernel update.
// (F_a, M_b): what the "b" side of a bond needs, stored as
// (F.x, F.y, M.x, M.y, F.z, M.z) so each (x, y) is an aligned fp32 pair.
template <class R> struct __align__(2 * sizeof(R)) Rec6 {
  R f[6];
};
template <class R> __device__ __forceinline__ Rec6<R> rec6(V3<R> F, V3<R> M) {
  return Rec6<R>{{F.x, F.y, M.x, M.y, F.z, M.z}};
}
// Slot sums (Eq. 25-26): a -axis slot adds (-F_a, M_b) of its record, a
// +axis slot (F_a, M_a) of the voxel's own bond.
template <class R> __device__ __forceinline__ void slot_minus(V3<R>& F, V3<R>& M, const Rec6<R>& r) {
  F = F - mk(r.f[0], r.f[1], r.f[4]);
  M = M + mk(r.f[2], r.f[3], r.f[5]);
}
template <class R> __device__ __forceinline__ void slot_plus(V3<R>& F, V3<R>& M, V3<R> Fo, V3<R> Mo) {
  F = F + Fo;
  M = M + Mo;
}
__device__ __forceinline__ void slot_minus(V3<float>& F, V3<float>& M, const Rec6<float>& r) {
  const f2_t fxy = sub2(f2pk(F.x, F.y), f2pk(r.f[0], r.f[1]));
  const f2_t mxy = add2(f2pk(M.x, M.y), f2pk(r.f[2], r.f[3]));
  F = mk(f2lo(fxy), f2hi(fxy), F.z - r.f[4]);
  M = mk(f2lo(mxy), f2hi(mxy), M.z + r.f[5]);
}
__device__ __forceinline__ void slot_plus(V3<float>& F, V3<float>& M, V3<float> Fo, V3<float> Mo) {
  const f2_t fxy = add2(f2pk(F.x, F.y), f2pk(Fo.x, Fo.y));
  const f2_t mxy = add2(f2pk(M.x, M.y), f2pk(Mo.x, Mo.y));
  F = mk(f2lo(fxy), f2hi(fxy), F.z + Fo.z);
  M = mk(f2lo(mxy), f2hi(mxy), M.z + Mo.z);
}
template <class R> struct FusedArgs {
  typename VT<R>::R4* opos;
  typename VT<R>::R4* oquat;
  typename VT<R>::R4* omom;
  typename VT<R>::R2* oang;
  const uint32_t* ext_of_local;
  int ty;           // rows per block
  int sx;           // planes per segment
  int p0, p1;       // local planes to update [p0, p1)
  int p0b, p1b;     // a second range, for blocks >= nblk0 (a slab's two boundary planes)
  int nblk0;
  int zchunks;      // z chunks of blockDim voxels (1 for nz <= 256)
  int ntiles_y;
  int nplanes;      // planes in the local box
};

#ifndef VX_PF_DIST
#define VX_PF_DIST 1
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}


// Thread k's +z neighbour is thread k+1's own voxel: a warp shuffle of its
// registers; lane 31 takes it from the next warp's lane 0 through shared
// memory (written before the previous row's barrier).
template <class R> __device__ __forceinline__ VS<R> vs_shfl_down(const VS<R>& s) {
  constexpr unsigned F = 0xffffffffu;
  VS<R> o;
  o.p.x = __shfl_down_sync(F, s.p.x, 1); o.p.y = __shfl_down_sync(F, s.p.y, 1);
  o.p.z = __shfl_down_sync(F, s.p.z, 1); o.p.w = __shfl_down_sync(F, s.p.w, 1);
  o.q.x = __shfl_down_sync(F, s.q.x, 1); o.q.y = __shfl_down_sync(F, s.q.y, 1);
  o.q.z = __shfl_down_sync(F, s.q.z, 1); o.q.w = __shfl_down_sync(F, s.q.w, 1);
  o.mo.x = __shfl_down_sync(F, s.mo.x, 1); o.mo.y = __shfl_down_sync(F, s.mo.y, 1);
  o.mo.z = __shfl_down_sync(F, s.mo.z, 1); o.mo.w = __shfl_down_sync(F, s.mo.w, 1);
  o.an.x = __shfl_down_sync(F, s.an.x, 1); o.an.y = __shfl_down_sync(F, s.an.y, 1);
  return o;
}

template <class R, bool COLLIDE, bool ZC>
__global__ void __launch_bounds__(256, sizeof(R) == 4 ? 2 : 1) k_step_fused(Dev<R> d, FusedArgs<R> a) {
  using R4 = typename VT<R>::R4;
  using R2 = typename VT<R>::R2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nzb = blockDim.x;
  // shared: xrec[ty][nzb], zrec[2][nzb] (Rec6), edge[2][nzb / 32] (VS: lane 0's
  // next-row voxel for lane 31 of the warp below)
  Rec6<R>* xrec = reinterpret_cast<Rec6<R>*>(smem_raw);
  Rec6<R>* zrec = xrec + (size_t)a.ty * nzb;
  VS<R>* edge = reinterpret_cast<VS<R>*>(zrec + 2 * (size_t)nzb);
  Rec6<R>* yrec = reinterpret_cast<Rec6<R>*>(edge + 2 * (nzb / 32));   // thread-private -y slot
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = nzb >> 5;
#ifdef VX_CHECKED
  // row tags of the zrec / edge slots (fused_smem reserves them)
  volatile int* ztag = reinterpret_cast<volatile int*>(yrec + nzb);
  volatile int* etag = ztag + 2 * nzb;
  for (int q = threadIdx.x; q < 2 * nzb + 2 * nwarp; q += nzb) ztag[q] = -1;
  __syncthreads();
#endif

  // z chunks of blockDim voxels (nz > 256): chunk zc covers k in [kz0, kz0 + nzb)
  const int tk = threadIdx.x;
  int bid = blockIdx.x, p0 = a.p0, p1 = a.p1;
  if (bid >= a.nblk0) { bid -= a.nblk0; p0 = a.p0b; p1 = a.p1b; }
  int kz0 = 0;
  if constexpr (ZC) {   // nz > 256
    const int zc = bid % a.zchunks;
    bid /= a.zchunks;
    kz0 = zc * nzb;
  }
  const int k = kz0 + tk;
  const bool act = k < (int)d.nz;
  const R kf = floor_base(d, (uint32_t)k);   // once per thread: k is fixed
  const int tile = bid % a.ntiles_y;
  const int seg = bid / a.ntiles_y;
  const int j0 = tile * a.ty;
  const int j1 = min(j0 + a.ty, (int)d.ny);
  const int i0 = p0 + seg * a.sx;
  const int i1 = min(i0 + a.sx, p1);
  const uint32_t sx = d.sx, nz = d.nz;
  const int ny = (int)d.ny;
  const R dT = (R)d.clk->dT;
  R vmax = R(0);
  auto idx = [&](int i, int j) { return (uint32_t)i * sx + (uint32_t)j * nz + (uint32_t)k; };

  // -x slots of plane i0: the +x bonds of plane i0 - 1 (halo, recomputed); the
  // next row's two voxels are loaded before this row's bond is evaluated
  if (act) {
    if (i0 > 0) {
      VS<R> pa = ldv(d, idx(i0 - 1, j0));
      VS<R> pb = ldv(d, idx(i0, j0));
      for (int j = j0; j < j1; ++j) {
        VS<R> na = pa, nb = pb;
        if (j + 1 < j1) {
          na = ldv(d, idx(i0 - 1, j + 1));
          nb = ldv(d, idx(i0, j + 1));
        }
        Rec6<R> r{};
        if (meta_of(pa.p.w) & nb_bit(1)) {
          const AFrame<R> f = a_frame(d, pa);
          V3<R> Fa, Ma, Mb;
          bond_eval<0>(d, f.Ra, pa.q, f.ua, f.Va, f.wa, f.mat, pb, dT, Fa, Ma, Mb);
          r = rec6(Fa, Mb);
        }
        xrec[(size_t)(j - j0) * nzb + tk] = r;
        pa = na;
        pb = nb;
      }
    } else {
      for (int j = j0; j < j1; ++j) xrec[(size_t)(j - j0) * nzb + tk] = Rec6<R>{};
    }
  }

  // zrec / edge buffer parity: a row counter carried across planes, so two
  // consecutive rows never share a buffer even when a tile has an odd number of
  // rows (the last row of plane i and the first of plane i+1 are adjacent)
  int rc = 0;
  for (int i = i0; i < i1; ++i) {
    VS<R> va, vb;    // ping-pong: this row's voxel and the next row's
    Rec6<R>& ry = yrec[tk];   // -y slot record of the current row: +y bond of the row below
    ry = Rec6<R>{};
    if (act) {
      va = ldv(d, idx(i, j0));
      if (j0 > 0) {   // halo row j0 - 1: its +y bond only
        const VS<R> vh = ldv(d, idx(i, j0 - 1));
        if (meta_of(vh.p.w) & nb_bit(3)) {
          const AFrame<R> f = a_frame(d, vh);
          V3<R> Fa, Ma, Mb;
          bond_eval<1>(d, f.Ra, vh.q, f.ua, f.Va, f.wa, f.mat, va, dT, Fa, Ma, Mb);
          ry = rec6(Fa, Mb);
        }
      }
    }
    // One row: voxel (i, j, k) in `cur`; loads row j+1's voxel into `nxt`.  One
    // block barrier: the -z slot (thread k-1's +z bond) goes through zrec[par].
    // FULL (a warp-uniform compile-time flag): every lane is an active, filled,
    // non-fixed voxel with all four x/y neighbours -- the interior of a solid;
    // the per-lane tests of those conditions and their branches drop out.
    auto row = [&](auto full, int j, const VS<R>& cur, VS<R>& nxt, int par) {
      constexpr bool FULL = decltype(full)::value;
      const uint32_t meta = (FULL || act) ? meta_of(cur.p.w) : 0u;
      const uint32_t id = idx(i, j);
      if (FULL || (act && (j + 1 < j1 || (meta & nb_bit(3)))))
        nxt = ldv(d, id + nz);
      VS<R> vx;
      if (FULL || (meta & nb_bit(1))) vx = ldv(d, id + sx);
      // the +x row VX_PF_DIST rows ahead (first touch: HBM) into L2, continuing into the
      // next plane of the segment at the end of the tile
      if (FULL || act) {
        int jj = j + VX_PF_DIST, ii = i + 1;
        if (jj >= j1) { jj -= j1 - j0; ++ii; }
        if (ii < a.nplanes && (ii == i + 1 || i + 1 < i1)) {
          const uint32_t f = idx(ii, jj);
          prefetch_l2(d.pos + f);
          prefetch_l2(d.quat + f);
          prefetch_l2(d.mom + f);
          prefetch_l2(d.ang + f);
        }
      }
      VS<R> vz = vs_shfl_down(cur);
      if (lane == 31 && (meta & nb_bit(5))) {   // the last lane of the block: the next chunk's
        if (j > j0 && (!ZC || warp + 1 < nwarp)) {
          VX_CHECKED_ONLY(__nanosleep(((unsigned)(warp * 977 + rc * 131)) % 1500u));
          vz = edge[(par ^ 1) * nwarp + warp + 1];
          VX_CHK(etag[(par ^ 1) * nwarp + warp + 1] == rc - 1, 3);
        } else {
          vz = ldv(d, id + 1);
        }
      }
      V3<R> FX{}, MX{}, BX{}, FY{}, MY{}, BY{}, FZ{}, MZ{}, BZ{};
      if (FULL || (meta & M_FILLED)) {
        const AFrame<R> f = a_frame(d, cur);
        if (meta & nb_bit(5)) bond_eval<2>(d, f.Ra, cur.q, f.ua, f.Va, f.wa, f.mat, vz, dT, FZ, MZ, BZ);
        if (FULL || (meta & nb_bit(1)))
          bond_eval<0>(d, f.Ra, cur.q, f.ua, f.Va, f.wa, f.mat, vx, dT, FX, MX, BX);
        if (FULL || (meta & nb_bit(3)))
          bond_eval<1>(d, f.Ra, cur.q, f.ua, f.Va, f.wa, f.mat, nxt, dT, FY, MY, BY);
      }
      if (lane == 0 && warp > 0 && (FULL || act) && j + 1 < j1) {
        edge[par * nwarp + warp] = nxt;
        VX_CHECKED_ONLY(__threadfence_block(); etag[par * nwarp + warp] = rc);
      }
      Rec6<R>* zr = zrec + (size_t)par * nzb;
      if (FULL || act) {
        zr[tk] = rec6(FZ, BZ);
        VX_CHECKED_ONLY(__threadfence_block(); ztag[par * nzb + tk] = rc);
      }
      // the first lane of a later z chunk: its -z bond belongs to the chunk below,
      // recomputed here (halo)
      Rec6<R> zlo{};
      if (ZC && tk == 0 && kz0 > 0 && (meta & nb_bit(4))) {
        const VS<R> vl = ldv(d, id - 1);
        const AFrame<R> f = a_frame(d, vl);
        V3<R> Fa, Ma, Mb;
        bond_eval<2>(d, f.Ra, vl.q, f.ua, f.Va, f.wa, f.mat, cur, dT, Fa, Ma, Mb);
        zlo = rec6(Fa, Mb);
      }
      // K4's slot order -x, +x, -y, +y | -z, +z: the first four before the barrier
      Rec6<R>& xr = xrec[(size_t)(j - j0) * nzb + tk];
      V3<R> F = mk(R(0), R(0), R(0)), M = F;
      if (FULL || (meta & nb_bit(0))) slot_minus(F, M, xr);
      if (FULL || (meta & nb_bit(1))) slot_plus(F, M, FX, MX);
      if (FULL || (meta & nb_bit(2))) slot_minus(F, M, ry);
      if (FULL || (meta & nb_bit(3))) slot_plus(F, M, FY, MY);
      if (FULL || (act && (meta & M_FILLED))) xr = rec6(FX, BX);
      ry = rec6(FY, BY);
      __syncthreads();
      if (!FULL && !act) return;
      VX_CHK(i >= p0 && i < p1, 7);
      if (FULL || (meta & (M_FILLED | M_FIXED)) == M_FILLED) {
#ifdef VX_CHECKED
        if ((meta & nb_bit(4)) && tk > 0) {   // widen the window of a lapping writer, then check
          // (longest after a plane's last row: the next write to this slot after it
          // is the next plane's first row, with no barrier of its own in between)
          if (lane == 0) __nanosleep(j == j1 - 1 ? 20000u : ((unsigned)(warp * 613 + rc * 97)) % 2000u);
          const Rec6<R> zz = zr[tk - 1];
          __threadfence_block();
          VX_CHK(ztag[par * nzb + tk - 1] == rc, 2);
          (void)zz;
        }
#endif
        if (meta & nb_bit(4)) slot_minus(F, M, (!ZC || tk > 0) ? zr[tk - 1] : zlo);
        if (meta & nb_bit(5)) slot_plus(F, M, FZ, MZ);
        const R v = finish_voxel<R, COLLIDE>(d, id, kf, cur, meta, F, M, a.opos, a.oquat, a.omom,
                                             a.oang, a.ext_of_local);
        vmax = fmax(vmax, v);
      } else if (meta & M_FILLED) {   // fixed: copied through unchanged
        st_stream(a.opos + id, cur.p);
        st_stream(a.oquat + id, cur.q);
        st_stream(a.omom + id, cur.mo);
        st_stream(a.oang + id, cur.an);
      } else {
        st_stream(a.opos + id, cur.p);   // empty cell: meta only
      }
    };
    constexpr uint32_t kXY = nb_bit(0) | nb_bit(1) | nb_bit(2) | nb_bit(3);
    auto is_full = [&](const VS<R>& v) {
      const uint32_t m = act ? meta_of(v.p.w) : 0u;
      return __all_sync(0xffffffffu, (m & (M_FILLED | M_FIXED | kXY)) == (M_FILLED | kXY));
    };
#ifdef VX_RACE_OLDPARITY   // the round-1 parity (restarts per plane): the probe must catch it
#define VX_PAR(j) (((j) - j0) & 1)
#else
#define VX_PAR(j) (rc & 1)
#endif
    for (int j = j0; j < j1;) {
      if (is_full(va)) {
        row(std::true_type{}, j, va, vb, VX_PAR(j));
        ++rc;
        ++j;
      } else {
        row(std::false_type{}, j, va, vb, VX_PAR(j));
        ++rc;
        ++j;
      }
      va = vb;
    }
#undef VX_PAR
  }
  if constexpr (COLLIDE) budget_max(d, vmax);
}

template <class R> size_t fused_smem(int ty, int nzb) {
  return sizeof(Rec6<R>) * ((size_t)ty * nzb + 3 * (size_t)nzb) + 2 * (size_t)(nzb / 32) * sizeof(VS<R>)
#ifdef VX_CHECKED
         + sizeof(int) * (2 * (size_t)nzb + 2 * (size_t)(nzb / 32))
#endif
      ;
}

// ------------------------------------------------------------------ K5 broadphase
// Surface table.  Every surface voxel of the whole lattice (all slabs) has a
// global surface index s, ascending in global box id gbox[s] (x-slowest), so
// each slab's surface voxels are one contiguous segment.  Each step the slabs
// pack their segment's state S_n into ss (ss[2s] = pos, ss[2s+1] = mom) and,
// over NCCL, broadcast it to every rank; the broadphase and the contact loads
// then read only ss, so a slab sees partners owned by any other slab (SURVEY
// §8f f3) and the arithmetic is the same for every slab count.
template <class R>
__global__ void __launch_bounds__(256) k_surf_pack(Dev<R> d, const unsigned* gbox, int s0, int s1,
                                                  typename VT<R>::R4* ss) {
  const int s = s0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= s1) return;
  const unsigned li = gbox[s] - (unsigned)d.xl0 * d.sx;
  ss[2 * s] = d.pos[li];
  ss[2 * s + 1] = d.mom[li];
}

// One CTA (1024 threads), gated by clk->rebuild.  All S surface voxels are
// hashed by cell floor(D / h), h >= cutoff; for the rows [r0, r1) (this
// rank's segment, or every row in one process) each partner with
// |D_a - D_b| < cutoff and lattice Manhattan distance > 3 goes into a
// CSR of global surface indices, each row sorted ascending (deterministic).
struct BroadArgs {
  const unsigned* gbox;   // S global box ids, ascending
  int S;                  // surface voxels of the whole lattice
  int r0, r1;             // rows built here
  int4* cellh;            // per surface voxel: cell x,y,z and hash
  int* bcount;            // H
  int* bstart;            // H + 1
  int* bitems;            // S
  int* rowptr;            // S + 1 (rows outside [r0, r1) are empty)
  int* col;               // cap
  long long cap;
  int H;                  // power of two
  Clock* clk;
  int batch_stride;       // planes per batched scene (0: one scene); no cross-scene pairs
  int batch_stride_z;     // layers per z-stacked batched scene (0: none)
  int batch_stride_y;     // rows per y-stacked batched scene (0: none)
  const int4* sijk;       // S lattice coordinates (i, j, k) of the surface entries
};

__device__ __forceinline__ int cell_hash(int x, int y, int z, int H) {
  unsigned h = (unsigned)x * 73856093u ^ (unsigned)y * 19349663u ^ (unsigned)z * 83492791u;
  return (int)(h & (unsigned)(H - 1));
}

// In-place exclusive scan of a[0..n) by one CTA of 1024 threads; a[n] = total.
__device__ void cta_exscan(int* a, int n) {
  __shared__ int part[1024];
  const int T = blockDim.x, t = threadIdx.x;
  const int chunk = (n + T - 1) / T;
  const int b = min(n, t * chunk), e = min(n, b + chunk);
  int s = 0;
  for (int i = b; i < e; ++i) s += a[i];
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < T; off <<= 1) {
    int v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int run = part[t] - s;
  for (int i = b; i < e; ++i) {
    int v = a[i];
    a[i] = run;
    run += v;
  }
  if (t == T - 1) a[n] = part[T - 1];
  __syncthreads();
}

// global box id -> lattice indices (box order: x slowest, z fastest)
template <class R>
__device__ __forceinline__ void box_ijk(const Dev<R>& d, unsigned g, int& i, int& j, int& k) {
  i = (int)(g / d.sx);
  const unsigned r = g - (unsigned)i * d.sx;
  j = (int)(r / d.nz);
  k = (int)(r - (unsigned)j * d.nz);
}

// Partners of surface voxel s (global surface indices u != s in the 27 cells
// around it with |D_s - D_u| < cutoff and lattice Manhattan distance > 3):
// counted (FILL = false) or written to col[base..) and sorted ascending.
// BP_LANES lanes share a row: lane c queries the cells c, c + L, ... of the 27
// around it (dz, dy, dx order).  The count pass sums the lanes' counts; the
// fill pass writes each lane's partners at its exclusive prefix and lane 0
// sorts the row ascending, so the row is the same set in the same order for
// any lane split (deterministic).  All lanes of a warp call this together.
constexpr int BP_LANES = 8;
template <bool FILL, class R>
__device__ __forceinline__ int bp_row(const Dev<R>& d, const BroadArgs& b,
                                      const typename VT<R>::R4* ss, int s, bool act, int c, R cutoff2,
                                      int base) {
  using R4 = typename VT<R>::R4;
  int cnt = 0;
  int4 cs = make_int4(0, 0, 0, 0), a = cs;
  R4 pa{};
  if (act) {
    cs = b.cellh[s];
    a = b.sijk[s];
    pa = ss[2 * s];
  }
  // the lane's candidates, twice: count, then (FILL) write at the prefix
  auto scan = [&](bool write, int at) {
    int n = 0;
    for (int ci = c; act && ci < 27; ci += BP_LANES) {
      const int cx = cs.x + ci % 3 - 1, cy = cs.y + (ci / 3) % 3 - 1, cz = cs.z + ci / 9 - 1;
      const int hh = cell_hash(cx, cy, cz, b.H);
      for (int q = b.bstart[hh]; q < b.bstart[hh + 1]; ++q) {
        const int u = b.bitems[q];
        const int4 cu = b.cellh[u];
        if (u == s || cu.x != cx || cu.y != cy || cu.z != cz) continue;
        const int4 o = b.sijk[u];
        if (abs(a.x - o.x) + abs(a.y - o.y) + abs(a.z - o.z) <= 3) continue;
        if (b.batch_stride && a.x / b.batch_stride != o.x / b.batch_stride) continue;
        if (b.batch_stride_z && a.z / b.batch_stride_z != o.z / b.batch_stride_z) continue;
        if (b.batch_stride_y && a.y / b.batch_stride_y != o.y / b.batch_stride_y) continue;
        const R4 pb = ss[2 * u];
        const R rx = d.l * (R)(a.x - o.x) + (pa.x - pb.x);
        const R ry = d.l * (R)(a.y - o.y) + (pa.y - pb.y);
        const R rz = d.l * (R)(a.z - o.z) + (pa.z - pb.z);
        if (rx * rx + ry * ry + rz * rz >= cutoff2) continue;
        if (write && at + n < b.cap) b.col[at + n] = u;
        ++n;
      }
    }
    return n;
  };
  const int lane = threadIdx.x & 31, g0 = lane & ~(BP_LANES - 1);
  const unsigned gm = BP_LANES == 32 ? 0xffffffffu : (((1u << (BP_LANES & 31)) - 1u) << g0);   // this row's lanes
  cnt = scan(false, 0);
  if (!FILL) {
#pragma unroll
    for (int o = BP_LANES / 2; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    return cnt;
  }
  // exclusive prefix of the lane counts within the row's lanes
  int pre = cnt;
#pragma unroll
  for (int o = 1; o < BP_LANES; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, pre, o);
    if ((lane & (BP_LANES - 1)) >= o) pre += v;
  }
  const int tot = __shfl_sync(0xffffffffu, pre, g0 + BP_LANES - 1);
  scan(true, base + pre - cnt);
  __syncwarp(gm);
  if (act && c == 0 && base + tot <= b.cap) {   // sort the row by partner index (deterministic)
    for (int x = base + 1; x < base + tot; ++x) {
      const int v = b.col[x];
      int y = x - 1;
      while (y >= base && b.col[y] > v) { b.col[y + 1] = b.col[y]; --y; }
      b.col[y + 1] = v;
    }
  }
  return tot;
}

// Cooperative launch over the whole GPU (grid-wide barriers between phases),
// 1024 threads per CTA; every CTA returns at once unless this step rebuilds.
// The two scans (bucket starts, row pointers) run in CTA 0.
template <class R>
__device__ __forceinline__ void broadphase_phases(const Dev<R>& d, const BroadArgs& b,
                                                  const typename VT<R>::R4* ss, double ox, double oy,
                                                  double oz, R h, R cutoff2, cg::grid_group& g) {
  using R4 = typename VT<R>::R4;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int x = tid; x < b.H; x += nth) b.bcount[x] = 0;
  g.sync();
  for (int s = tid; s < b.S; s += nth) {
    const int4 ijk = b.sijk[s];
    const int i = ijk.x, j = ijk.y, k = ijk.z;
    const R4 p = ss[2 * s];
    const R Dx = (R)(ox + d.l_d * ((double)i + 0.5)) + p.x;
    const R Dy = (R)(oy + d.l_d * ((double)j + 0.5)) + p.y;
    const R Dz = (R)(oz + d.l_d * ((double)k + 0.5)) + p.z;
    const int cx = (int)floor(Dx / h), cy = (int)floor(Dy / h), cz = (int)floor(Dz / h);
    const int hh = cell_hash(cx, cy, cz, b.H);
    b.cellh[s] = make_int4(cx, cy, cz, hh);
    atomicAdd(&b.bcount[hh], 1);
  }
  g.sync();
  if (blockIdx.x == 0) {
    for (int x = threadIdx.x; x < b.H; x += blockDim.x) b.bstart[x] = b.bcount[x];
    __syncthreads();
    cta_exscan(b.bstart, b.H);
    for (int x = threadIdx.x; x < b.H; x += blockDim.x) b.bcount[x] = 0;
  }
  g.sync();
  for (int s = tid; s < b.S; s += nth) {
    const int hh = b.cellh[s].w;
    b.bitems[b.bstart[hh] + atomicAdd(&b.bcount[hh], 1)] = s;
  }
  g.sync();
  // BP_LANES lanes per row; whole warps iterate together (shuffles in bp_row)
  const int lane = threadIdx.x & 31;
  const long long nrl = (long long)b.S * BP_LANES;
  for (long long t0 = tid - lane; t0 < nrl; t0 += nth) {
    const long long t = t0 + lane;
    const int s = (int)(t / BP_LANES), c = (int)(t % BP_LANES);
    const bool act = t < nrl && s >= b.r0 && s < b.r1;
    const int n = bp_row<false>(d, b, ss, s, act, c, cutoff2, 0);
    if (t < nrl && c == 0) b.rowptr[s] = act ? n : 0;
  }
  g.sync();
  if (blockIdx.x == 0) {
    cta_exscan(b.rowptr, b.S);
    if (threadIdx.x == 0) {
      const long long tot = b.rowptr[b.S];
      if (tot > b.cap) d.clk->overflow = 1;
      d.clk->npairs = tot;          // half-edges of the rows built here
      d.clk->rebuilds += 1;
    }
  }
  g.sync();
  for (long long t0 = tid - lane; t0 < nrl; t0 += nth) {
    const long long t = t0 + lane;
    const int s = (int)(t / BP_LANES), c = (int)(t % BP_LANES);
    const bool act = t < nrl && s >= b.r0 && s < b.r1;
    bp_row<true>(d, b, ss, s, act, c, cutoff2, act ? b.rowptr[s] : 0);
  }
}
template <class R>
__global__ void __launch_bounds__(1024, 1) k_broadphase(Dev<R> d, BroadArgs b, const typename VT<R>::R4* ss,
                                                     double ox, double oy, double oz, R h, R cutoff2) {
  if (!d.clk->rebuild) return;
  cg::grid_group g = cg::this_grid();
  broadphase_phases(d, b, ss, ox, oy, oz, h, cutoff2, g);
}

// ------------------------------------------------------------------ contact
// Penalty law of reading R16: F_on_a = max(0, k_c q - c_c v_n) n,
// q = r_a + r_b - |D_a - D_b|.  Rows [r0, r1) are one slab's segment; the load
// goes to that slab's cf at the voxel's local id.
// Contact loads of surface row s (row a7): the pair law over its CSR partners.
// CONTACT_LANES lanes share a row: lane c takes partners c, c + L, c + 2L, ...
// of the ascending partner list, and the L partial sums are combined by a fixed
// butterfly -- deterministic, the same on every engine and slab count (one
// kernel), and equal to the oracle's ascending sum up to rounding.  The lattice
// coordinates of surface entries come from a table (sijk), not divisions.
constexpr int CONTACT_LANES = 8;
template <class R>
__global__ void __launch_bounds__(256) k_contact(Dev<R> d, const unsigned* gbox, const int4* sijk,
                                                 const typename VT<R>::R4* ss, int r0, int r1,
                                                 const int* rowptr, const int* col, R zeta_col) {
  using R4 = typename VT<R>::R4;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = r0 + t / CONTACT_LANES, c = t % CONTACT_LANES;
  const bool row = s < r1;
  V3<R> F = mk(R(0), R(0), R(0));
  if (row) {
    const int4 a = sijk[s];
    const R4 pa = ss[2 * s];
    const MatC<R>& ma = d.mat[meta_of(pa.w) & M_MAT];
    const R4 moa = ss[2 * s + 1];
    const R dT = (R)d.clk->dT;
    const R ra = d.half_l * (R(1) + ma.alpha * dT);
    // after a pair-list overflow the row pointers exceed the list (VX_ERR_STATE is
    // reported at the end of vx_step): never read past it
    const int q1 = d.clk->overflow ? 0 : rowptr[s + 1];
    for (int q = rowptr[s] + c; q < q1; q += CONTACT_LANES) {
      const int u = col[q];
      const int4 b = sijk[u];
      const R4 pb = ss[2 * u];
      const MatC<R>& mb = d.mat[meta_of(pb.w) & M_MAT];
      const R rb = d.half_l * (R(1) + mb.alpha * dT);
      const V3<R> dd = mk(d.l * (R)(a.x - b.x) + (pa.x - pb.x), d.l * (R)(a.y - b.y) + (pa.y - pb.y),
                          d.l * (R)(a.z - b.z) + (pa.z - pb.z));
      const R dist = vx_sqrt(dot(dd, dd));
      const R pen = ra + rb - dist;
      if (!(pen > R(0))) continue;
      V3<R> n;
      // coincident centres (reading R16: closer than 1e-6 l): +z for the
      // voxel with the lower external id (x-fastest order = lexicographic
      // (k, j, i)), -z for the other
      if (dist > R(1e-6) * d.l) n = (R(1) / dist) * dd;
      else n = mk(R(0), R(0), (a.z != b.z ? a.z < b.z : a.y != b.y ? a.y < b.y : a.x < b.x) ? R(1) : R(-1));
      const R4 mob = ss[2 * u + 1];
      const V3<R> Va = ma.inv_m * mk(moa.x, moa.y, moa.z);
      const V3<R> Vb = mb.inv_m * mk(mob.x, mob.y, mob.z);
      const R vn = dot(Va - Vb, n);
      const R kc = R(2) * ma.kc * mb.kc / (ma.kc + mb.kc);
      const R cc = R(2) * zeta_col * vx_sqrt(fmin(ma.m, mb.m) * kc);
      R f = kc * pen - cc * vn;
      if (f < R(0)) f = R(0);
      F = F + f * n;
    }
  }
#pragma unroll
  for (int o = CONTACT_LANES / 2; o > 0; o >>= 1) {
    F.x = F.x + __shfl_xor_sync(0xffffffffu, F.x, o);
    F.y = F.y + __shfl_xor_sync(0xffffffffu, F.y, o);
    F.z = F.z + __shfl_xor_sync(0xffffffffu, F.z, o);
  }
  if (row && c == 0) d.cf[gbox[s] - (unsigned)d.xl0 * d.sx] = R4{F.x, F.y, F.z, R(0)};
}

// ------------------------------------------------------------------ state I/O
// Rest site coordinate o + l (i + 1/2), rounded as two separate fp64
// operations (no FMA contraction), i.e. exactly as a caller forms it.
__device__ __forceinline__ double site(double o, double l, long long i) {
  return __dadd_rn(o, __dmul_rn(l, (double)i + 0.5));
}

// External arrays (fp64) <-> device state.  box_of_ext[e] = global box id of
// external voxel e; local id = box - box_base when within [0, nloc).
template <class R>
__global__ void k_scatter_state(Dev<R> d, const long long* box_of_ext, long long N,
                                long long box_base, const double* pos, const double* quat,
                                const double* lin, const double* ang, const uint8_t* latch,
                                double ox, double oy, double oz) {
  using R4 = typename VT<R>::R4;
  using R2 = typename VT<R>::R2;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  const long long g = box_of_ext[e];
  const long long li = g - box_base;
  if (li < 0 || li >= (long long)d.nloc) return;
  const long long nyz = (long long)d.ny * d.nz;
  const long long i = g / nyz, j = (g / d.nz) % d.ny, k = g % d.nz;
  const double l = d.l_d;
  R4 p = d.pos[li];
  if (pos) {
    p.x = (R)(pos[3 * e] - site(ox, l, i));
    p.y = (R)(pos[3 * e + 1] - site(oy, l, j));
    p.z = (R)(pos[3 * e + 2] - site(oz, l, k));
  }
  if (latch) {
    uint32_t m = meta_of(p.w);
    m = latch[e] ? (m | M_LATCH) : (m & ~M_LATCH);
    p.w = meta_as(R(0), m);
  }
  d.pos[li] = p;
  if (quat) d.quat[li] = R4{(R)quat[4 * e + 1], (R)quat[4 * e + 2], (R)quat[4 * e + 3], (R)quat[4 * e]};
  R4 mo = d.mom[li];
  R2 an = d.ang[li];
  if (lin) { mo.x = (R)lin[3 * e]; mo.y = (R)lin[3 * e + 1]; mo.z = (R)lin[3 * e + 2]; }
  if (ang) { an.x = (R)ang[3 * e]; an.y = (R)ang[3 * e + 1]; mo.w = (R)ang[3 * e + 2]; }
  d.mom[li] = mo;
  d.ang[li] = an;
}

// Owned local range -> box-ordered fp64 SoA (14 components x nbox_global).
template <class R>
__global__ void k_pack_box(Dev<R> d, uint32_t beg, uint32_t end, long long box_base,
                           long long nbox, double* out, double ox, double oy, double oz) {
  const uint32_t li = beg + blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= end) return;
  const long long g = box_base + li;
  const long long nyz = (long long)d.ny * d.nz;
  const long long i = g / nyz, j = (g / d.nz) % d.ny, k = g % d.nz;
  const double l = d.l_d;
  const auto p = d.pos[li];
  const auto q = d.quat[li];
  const auto mo = d.mom[li];
  const auto an = d.ang[li];
  double v[14] = {site(ox, l, i) + (double)p.x, site(oy, l, j) + (double)p.y,
                  site(oz, l, k) + (double)p.z, (double)q.w, (double)q.x,
                  (double)q.y, (double)q.z, (double)mo.x, (double)mo.y, (double)mo.z,
                  (double)an.x, (double)an.y, (double)mo.w,
                  (meta_of(p.w) & M_LATCH) ? 1.0 : 0.0};
#pragma unroll
  for (int c = 0; c < 14; ++c) out[c * nbox + g] = v[c];
}

// box-ordered SoA -> external-order arrays
__global__ void k_box_to_ext(const double* box, long long nbox, const long long* box_of_ext,
                             long long N, double* pos, double* quat, double* lin, double* ang,
                             uint8_t* latch) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  const long long g = box_of_ext[e];
  for (int c = 0; c < 3; ++c) pos[3 * e + c] = box[c * nbox + g];
  for (int c = 0; c < 4; ++c) quat[4 * e + c] = box[(3 + c) * nbox + g];
  for (int c = 0; c < 3; ++c) lin[3 * e + c] = box[(7 + c) * nbox + g];
  for (int c = 0; c < 3; ++c) ang[3 * e + c] = box[(10 + c) * nbox + g];
  latch[e] = box[13 * nbox + g] != 0.0;
}

// Selected voxels (local ids, -1 = not owned) -> fp64 arrays.
template <class R>
__global__ void k_read_ids(Dev<R> d, const long long* lids, const long long* gids, long long n,
                           double* pos, double* quat, double* lin, double* ang,
                           uint8_t* latch, double ox, double oy, double oz) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const long long li = lids[e], g = gids[e];
  const long long nyz = (long long)d.ny * d.nz;
  const long long i = g / nyz, j = (g / d.nz) % d.ny, k = g % d.nz;
  const double l = d.l_d;
  const auto p = d.pos[li];
  const auto q = d.quat[li];
  const auto mo = d.mom[li];
  const auto an = d.ang[li];
  pos[3 * e] = site(ox, l, i) + (double)p.x;
  pos[3 * e + 1] = site(oy, l, j) + (double)p.y;
  pos[3 * e + 2] = site(oz, l, k) + (double)p.z;
  quat[4 * e] = q.w; quat[4 * e + 1] = q.x; quat[4 * e + 2] = q.y; quat[4 * e + 3] = q.z;
  lin[3 * e] = mo.x; lin[3 * e + 1] = mo.y; lin[3 * e + 2] = mo.z;
  ang[3 * e] = an.x; ang[3 * e + 1] = an.y; ang[3 * e + 2] = mo.w;
  latch[e] = (meta_of(p.w) & M_LATCH) ? 1 : 0;
}

// Owned-voxel gather (vx_read_state_owned): entries dst[e] of the output
// arrays from local id lid[e] (global box id gid[e]) of one slab.
template <class R>
__global__ void k_gather_owned(Dev<R> d, const long long* lid, const long long* gid, const long long* dst,
                               long long n, long long m, double* out, uint8_t* latch, double ox, double oy,
                               double oz) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const long long li = lid[e], g = gid[e], t = dst[e];
  const long long nyz = (long long)d.ny * d.nz;
  const long long i = g / nyz, j = (g / d.nz) % d.ny, k = g % d.nz;
  const double l = d.l_d;
  const auto p = d.pos[li];
  const auto q = d.quat[li];
  const auto mo = d.mom[li];
  const auto an = d.ang[li];
  double* pos = out;
  double* quat = out + m * 3;
  double* lin = out + m * 7;
  double* ang = out + m * 10;
  pos[3 * t] = site(ox, l, i) + (double)p.x;
  pos[3 * t + 1] = site(oy, l, j) + (double)p.y;
  pos[3 * t + 2] = site(oz, l, k) + (double)p.z;
  quat[4 * t] = q.w; quat[4 * t + 1] = q.x; quat[4 * t + 2] = q.y; quat[4 * t + 3] = q.z;
  lin[3 * t] = mo.x; lin[3 * t + 1] = mo.y; lin[3 * t + 2] = mo.z;
  ang[3 * t] = an.x; ang[3 * t + 1] = an.y; ang[3 * t + 2] = mo.w;
  latch[t] = (meta_of(p.w) & M_LATCH) ? 1 : 0;
}

// Merge static meta bits (material, filled, fixed, surface, ext, neighbours)
// with the dynamic latch bit.
template <class R>
__global__ void k_merge_meta(Dev<R> d, const uint32_t* meta_static, uint32_t n) {
  const uint32_t li = blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= n) return;
  auto p = d.pos[li];
  const uint32_t m = (meta_static[li] & ~M_LATCH) | (meta_of(p.w) & M_LATCH);
  p.w = meta_as(decltype(p.x)(0), m);
  d.pos[li] = p;
}

}  // namespace vx
