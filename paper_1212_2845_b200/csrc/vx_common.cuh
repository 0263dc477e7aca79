// vx_common.cuh -- device types, SoA layout and small vector/quaternion math
// for the voxel stepper (arXiv:1212.2845).  Product path: shares nothing with
// oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vx {

// ---------------------------------------------------------------- device checks
// The checked build (-DVX_CHECKED, libvoxsim_checked.so; build.py) bounds-checks
// every state load and store of the step kernels and tags the shared-memory
// records handed between threads (k_step_fused's -z record and edge row,
// k_step_fused_yz's -y ring and -z record) with the row that wrote them, so a
// consumer that finds another row's tag has caught a write-after-read race; it
// also delays the consumers of cross-warp handoffs to widen any such window.
// The first failed check is kept as (code << 32) | source line and vx_step
// reports it as VX_ERR_STATE.  Codes: 1 state load index, 2 -z record race,
// 3 edge-row race, 4 material index, 5 -y ring race (yz pass), 6 -z record
// race (yz pass), 7 state store outside the launch's planes.
// In normal builds VX_CHK compiles to nothing.
#ifdef VX_CHECKED
__device__ unsigned long long g_vx_chk = 0ULL;
#define VX_CHK(cond, code)                                                                      \
  do {                                                                                          \
    if (!(cond))                                                                                \
      atomicCAS(&::vx::g_vx_chk, 0ULL, ((unsigned long long)(code) << 32) | (unsigned)__LINE__); \
  } while (0)
#define VX_CHECKED_ONLY(x) x
#else
#define VX_CHK(cond, code) \
  do {                     \
  } while (0)
#define VX_CHECKED_ONLY(x)
#endif

// ---------------------------------------------------------------- layout
// Per-voxel state, box-indexed (internal id = ((i - xl0) * ny + j) * nz + k,
// x slowest so an x-slab and each x-plane is one contiguous range):
//   pos  R4 = (u.x, u.y, u.z, meta bits)   u = D - D_rest (displacement)
//   quat R4 = (x, y, z, w)   (CUDA member order; .w is the scalar part)
//   mom  R4 = (P.x, P.y, P.z, phi.x)
//   ang  R2 = (phi.y, phi.z)
// Bond records per axis a (bond (v, v+e_a) stored at v):
//   recA R4 = (Fa.x, Fa.y, Fa.z, Ma.x)
//   recB R4 = (Ma.y, Ma.z, Mb.x, Mb.y)
//   recC R  = Mb.z
// meta bits (uint32):
enum : uint32_t {
  M_MAT = 0xffu,          // material index (0-based)
  M_FILLED = 1u << 8,
  M_FIXED = 1u << 9,
  M_LATCH = 1u << 10,
  M_SURF = 1u << 11,
  M_EXT = 1u << 12,       // has an external force (fext array)
  M_NB_SHIFT = 16,        // 6 bits: -x,+x,-y,+y,-z,+z
};
__host__ __device__ constexpr uint32_t nb_bit(int slot) { return 1u << (M_NB_SHIFT + slot); }

template <class R> struct VT;
template <> struct VT<float> {
  using R4 = float4;
  using R2 = float2;
  using UB = unsigned int;          // bit pattern type for max-reductions
};
template <> struct VT<double> {
  using R4 = double4;
  using R2 = double2;
  using UB = unsigned long long;
};

__device__ __forceinline__ uint32_t meta_of(float w) { return __float_as_uint(w); }
__device__ __forceinline__ uint32_t meta_of(double w) {
  return (uint32_t)(unsigned long long)__double_as_longlong(w);
}
__device__ __forceinline__ float meta_as(float, uint32_t m) { return __uint_as_float(m); }
__device__ __forceinline__ double meta_as(double, uint32_t m) {
  return __longlong_as_double((long long)(unsigned long long)m);
}
__device__ __forceinline__ unsigned int rbits(float x) { return __float_as_uint(x); }
__device__ __forceinline__ unsigned long long rbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

// Per-material constants (host fp64, cast to R).
// (16-byte aligned, multiples of 4 scalars: loaded as 128-bit vectors)
template <class R> struct __align__(16) MatC {
  R m, inv_m, inv_I, dt_m, dt_I;  // dt_m = dt/m, dt_I = dt/I
  R mg;                           // m * g
  R cgt, cgr;                     // ground damping 2 zeta_g sqrt(m E l), 2 zeta_g sqrt(I G l^3/6)
  R kf, cfl;                      // floor stiffness E l and damping 2 zeta_col sqrt(m kf)
  R alpha, mu_s, mu_d;
  R kc;                           // contact stiffness E l
  R pad0, pad1;
};
// Per ordered material-pair (a, b) constants (Eq. 1-12, 34-35, 40).
// Laid out so (a1, a2) and (nb2, b2) are aligned pairs for the FP32x2 bond.
template <class R> struct __align__(16) PairC {
  R a1, a2, nb2, b2;              // nb2 = -b2
  R b1, b3;
  R alpha_mean;                   // (alpha_1 + alpha_2) / 2
  R ct2, ct4, cr2;                // c_t/2, c_t/4, c_r/2 with c_t = 2 zeta_b sqrt(m_min a1),
                                  // c_r = 2 zeta_b sqrt(I_min a2)
  R inv_m_b, inv_I_b;             // 1/m, 1/I of material b (damping velocities)
};

// ---------------------------------------------------------------- vec3
template <class R> struct V3 {
  R x, y, z;
};
template <class R> __device__ __forceinline__ V3<R> mk(R x, R y, R z) { return {x, y, z}; }
template <class R> __device__ __forceinline__ V3<R> operator+(V3<R> a, V3<R> b) {
  return {a.x + b.x, a.y + b.y, a.z + b.z};
}
template <class R> __device__ __forceinline__ V3<R> operator-(V3<R> a, V3<R> b) {
  return {a.x - b.x, a.y - b.y, a.z - b.z};
}
template <class R> __device__ __forceinline__ V3<R> operator*(R s, V3<R> a) {
  return {s * a.x, s * a.y, s * a.z};
}
template <class R> __device__ __forceinline__ V3<R> cross(V3<R> a, V3<R> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class R> __device__ __forceinline__ R dot(V3<R> a, V3<R> b) {
  return a.x * b.x + a.y * b.y + a.z * b.z;
}
template <class R> __device__ __forceinline__ R comp(V3<R> a, int i) {
  return i == 0 ? a.x : (i == 1 ? a.y : a.z);
}

// ---------------------------------------------------------------- explicit rounding
// Each helper rounds once, as written: the compiler may not fuse a product
// into a later sum (FMA contraction).  The frame and bond arithmetic is
// written with them, so every inlined copy -- a halo recomputation or a row of
// the fused sweep, K3 -- gives bit-identical results whatever code surrounds
// it (slab-count and launch-geometry invariance rest on this).
__device__ __forceinline__ float xmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float xadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float xsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float xfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double xfma(double a, double b, double c) { return __fma_rn(a, b, c); }
template <class R> __device__ __forceinline__ V3<R> xadd3(V3<R> a, V3<R> b) {
  return {xadd(a.x, b.x), xadd(a.y, b.y), xadd(a.z, b.z)};
}
template <class R> __device__ __forceinline__ V3<R> xsub3(V3<R> a, V3<R> b) {
  return {xsub(a.x, b.x), xsub(a.y, b.y), xsub(a.z, b.z)};
}
template <class R> __device__ __forceinline__ V3<R> xscale3(R s, V3<R> a) {
  return {xmul(s, a.x), xmul(s, a.y), xmul(s, a.z)};
}
template <class R> __device__ __forceinline__ V3<R> xfma3(R s, V3<R> a, V3<R> c) {   // s a + c
  return {xfma(s, a.x, c.x), xfma(s, a.y, c.y), xfma(s, a.z, c.z)};
}
template <class R> __device__ __forceinline__ V3<R> xcross(V3<R> a, V3<R> b) {
  return {xfma(a.y, b.z, xmul(-a.z, b.y)), xfma(a.z, b.x, xmul(-a.x, b.z)),
          xfma(a.x, b.y, xmul(-a.y, b.x))};
}
// a x + b y + c z, left to right
template <class R> __device__ __forceinline__ R xdot3(R a, R x, R b, R y, R c, R z) {
  return xfma(c, z, xfma(b, y, xmul(a, x)));
}

// Rotation matrix of a unit quaternion, split as R = I + Dm with the
// diagonal of Dm formed without cancellation (-2(y^2+z^2) ...).
template <class R> struct Rot {
  R m[3][3];   // full rotation matrix
  R dd[3];     // m[i][i] - 1
};
template <class R> __device__ __forceinline__ Rot<R> rotation(R w, R x, R y, R z) {
  Rot<R> r;
  const R two = R(2);
  r.dd[0] = xmul(-two, xfma(z, z, xmul(y, y)));
  r.dd[1] = xmul(-two, xfma(z, z, xmul(x, x)));
  r.dd[2] = xmul(-two, xfma(y, y, xmul(x, x)));
  r.m[0][0] = xadd(R(1), r.dd[0]);
  r.m[1][1] = xadd(R(1), r.dd[1]);
  r.m[2][2] = xadd(R(1), r.dd[2]);
  r.m[0][1] = xmul(two, xfma(-w, z, xmul(x, y)));
  r.m[0][2] = xmul(two, xfma(w, y, xmul(x, z)));
  r.m[1][0] = xmul(two, xfma(w, z, xmul(x, y)));
  r.m[1][2] = xmul(two, xfma(-w, x, xmul(y, z)));
  r.m[2][0] = xmul(two, xfma(-w, y, xmul(x, z)));
  r.m[2][1] = xmul(two, xfma(w, x, xmul(y, z)));
  return r;
}
template <class R> __device__ __forceinline__ V3<R> mul(const Rot<R>& r, V3<R> a) {
  return {xdot3(r.m[0][0], a.x, r.m[0][1], a.y, r.m[0][2], a.z),
          xdot3(r.m[1][0], a.x, r.m[1][1], a.y, r.m[1][2], a.z),
          xdot3(r.m[2][0], a.x, r.m[2][1], a.y, r.m[2][2], a.z)};
}
template <class R> __device__ __forceinline__ V3<R> mulT(const Rot<R>& r, V3<R> a) {
  return {xdot3(r.m[0][0], a.x, r.m[1][0], a.y, r.m[2][0], a.z),
          xdot3(r.m[0][1], a.x, r.m[1][1], a.y, r.m[2][1], a.z),
          xdot3(r.m[0][2], a.x, r.m[1][2], a.y, r.m[2][2], a.z)};
}

// ---------------------------------------------------------------- fp32 pairs
// sm_100's FP32x2 path: FADD2 / FMUL2 / FFMA2 perform two fp32 operations per
// instruction, each half rounded exactly like the scalar instruction.  A
// broadcast scalar, a swapped pair and a negated half are operand modifiers,
// so pairing (x, y) halves the issue slots of 2-vector work.  Pairs live in
// 64-bit registers: the halves of a loaded float4 / float2 are pairs already.
// (The compiler's float2 intrinsics __ffma2_rn / __fmul2_rn / __fadd2_rn give
// the same SASS; profiles/r14_experiments.md.)
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2pk(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2lo(f2_t r) {
  float lo;
  asm("mov.b64 {%0, _}, %1;" : "=f"(lo) : "l"(r));
  return lo;
}
__device__ __forceinline__ float f2hi(f2_t r) {
  float hi;
  asm("mov.b64 {_, %0}, %1;" : "=f"(hi) : "l"(r));
  return hi;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t bc2(float s) { return f2pk(s, s); }
__device__ __forceinline__ f2_t zero2() { return f2pk(0.f, 0.f); }

// fp32 rotation matrix packed for R v: column pairs (m0j, m1j), row 2 scalar.
struct RotP {
  f2_t c0, c1, c2;          // (m00, m10), (m01, m11), (m02, m12)
  float m20, m21, m22;
  float dd0, dd1, dd2;      // m_ii - 1, formed without cancellation
};
// Same formulas and operation order as rotation(): e.g. m10 = 2 (x y + w z),
// dd0 = -2 (y^2 + z^2); pairs Q1 = (x, y), Q2 = (z, w) of the quaternion.
__device__ __forceinline__ RotP rotation_p(float x, float y, float z, float w) {
  RotP r;
  const f2_t Q1 = f2pk(x, y);
  const f2_t nyx = f2pk(-y, x);
  // column 0: 2 (-(y y + z z), x y + w z)
  const f2_t t0 = mul2(fma2(f2pk(-z, w), bc2(z), mul2(nyx, bc2(y))), bc2(2.f));
  // column 1: 2 (x y - w z, -(x x + z z))
  const f2_t t1 = mul2(fma2(f2pk(-w, -z), bc2(z), mul2(nyx, bc2(-x))), bc2(2.f));
  // column 2: 2 (x z + w y, y z - w x); row 2: 2 (x z - w y, y z + w x)
  const f2_t xzyz = mul2(Q1, bc2(z));
  r.c2 = mul2(fma2(nyx, bc2(-w), xzyz), bc2(2.f));
  const f2_t r2 = mul2(fma2(nyx, bc2(w), xzyz), bc2(2.f));
  r.dd0 = f2lo(t0);
  r.dd1 = f2hi(t1);
  r.dd2 = xmul(-2.f, xfma(y, y, xmul(x, x)));
  r.c0 = add2(t0, f2pk(1.f, 0.f));
  r.c1 = add2(t1, f2pk(0.f, 1.f));
  r.m20 = f2lo(r2);
  r.m21 = f2hi(r2);
  r.m22 = xadd(1.f, r.dd2);
  return r;
}
// R a = a.x c0 + a.y c1 + a.z c2 (x, y packed)
__device__ __forceinline__ V3<float> mul(const RotP& r, V3<float> a) {
  const f2_t xy = fma2(r.c2, bc2(a.z), fma2(r.c1, bc2(a.y), mul2(r.c0, bc2(a.x))));
  return {f2lo(xy), f2hi(xy), xdot3(r.m20, a.x, r.m21, a.y, r.m22, a.z)};
}
// R^T a: one dot product per column
__device__ __forceinline__ V3<float> mulT(const RotP& r, V3<float> a) {
  return {xdot3(f2lo(r.c0), a.x, f2hi(r.c0), a.y, r.m20, a.z),
          xdot3(f2lo(r.c1), a.x, f2hi(r.c1), a.y, r.m21, a.z),
          xdot3(f2lo(r.c2), a.x, f2hi(r.c2), a.y, r.m22, a.z)};
}

// Cyclic permutation Pi of reading R5: world -> bond frame of axis AX.
template <int AX, class R> __device__ __forceinline__ V3<R> to_bond(V3<R> a) {
  if constexpr (AX == 0) return a;
  else if constexpr (AX == 1) return {a.y, a.z, a.x};
  else return {a.z, a.x, a.y};
}
template <int AX, class R> __device__ __forceinline__ V3<R> to_world(V3<R> a) {
  if constexpr (AX == 0) return a;
  else if constexpr (AX == 1) return {a.z, a.x, a.y};
  else return {a.y, a.z, a.x};
}

__device__ __forceinline__ float vx_atan2(float y, float x) { return atan2f(y, x); }
__device__ __forceinline__ double vx_atan2(double y, double x) { return atan2(y, x); }
__device__ __forceinline__ float vx_sqrt(float x) { return sqrtf(x); }
// 1/sqrt(x) for renormalising a unit quaternion: fp32 uses the hardware
// reciprocal square root (MUFU.RSQ, ~2 ulp: the factor is ~1 +- 1e-7 anyway)
__device__ __forceinline__ float vx_rnorm(float x) { return rsqrtf(x); }
__device__ __forceinline__ double vx_rnorm(double x) { return 1.0 / sqrt(x); }
__device__ __forceinline__ double vx_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ void vx_sincos(float a, float* s, float* c) { sincosf(a, s, c); }
__device__ __forceinline__ void vx_sincos(double a, double* s, double* c) { sincos(a, s, c); }
__device__ __forceinline__ bool vx_finite(float x) { return isfinite(x); }
__device__ __forceinline__ bool vx_finite(double x) { return isfinite(x); }

}  // namespace vx
