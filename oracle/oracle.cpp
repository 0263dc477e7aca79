/*
 * oracle.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain fp64 CPU stepper written step by step from the paper
 * (Hiller & Lipson, arXiv:1212.2845).  "P:n" = PAPER.md line n.
 * Ambiguous points take the readings of SURVEY.md §8(c):
 *   R1  F_z1 sign at P:194 read as -b1 Z2 - b2 theta_y2 (row 3 of Eq. 7).
 *   R3  the loads on the voxels are -[K]u (Eq. 13-24 negated).
 *   R4  voxel "1" of a bond is the voxel on the negative lattice side.
 *   R5  y/z bonds use the cyclic permutations (x,y,z)->(y,z,x) / (z,x,y).
 *   R6  orientation is a unit quaternion, world-frame increment (Eq. 30).
 *   R7  theta = 2 atan2(|v|, w) v/|v| with w >= 0.
 *   R8  I = m l^2 / 6.
 *   R9  dt = safety / (2 pi sqrt(max_b a1/m_min))     (Eq. 31-32, literal).
 *   R10 bond damping uses m_min, I_min of the bond (one coefficient).
 *   R11 rotational damping stiffness k_phi = a2.
 *   R12 ground damping: 2 zeta_g sqrt(m E l) V and 2 zeta_g sqrt(I G l^3/6) w.
 *   R14 floor: k_f = E l, radius (l/2)(1 + alpha dT), normal damping zeta_col.
 *   R15 friction sequencing as in SURVEY §8(c) step 4.5; zero lateral P before
 *       the position update.
 *   R16 self-collision law: penalty k_c q along the centre line plus normal
 *       damping, all pairs of surface voxels with lattice Manhattan > 3.
 * No blocking, fusion or reordering beyond the paper's two phases.
 */
#include "oracle.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

const double kPi = 3.14159265358979323846;

struct Vec3 {
  double x = 0, y = 0, z = 0;
};
Vec3 v3(double x, double y, double z) { Vec3 r; r.x = x; r.y = y; r.z = z; return r; }
Vec3 operator+(Vec3 a, Vec3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
Vec3 operator-(Vec3 a, Vec3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
Vec3 operator-(Vec3 a) { return v3(-a.x, -a.y, -a.z); }
Vec3 operator*(double s, Vec3 a) { return v3(s * a.x, s * a.y, s * a.z); }
double dot(Vec3 a, Vec3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
Vec3 cross(Vec3 a, Vec3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
double norm(Vec3 a) { return std::sqrt(dot(a, a)); }

struct Quat {
  double w = 1, x = 0, y = 0, z = 0;
};
/* Hamilton product */
Quat qmul(Quat a, Quat b) {
  Quat r;
  r.w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
  r.x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
  r.y = a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x;
  r.z = a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w;
  return r;
}
Quat qconj(Quat a) { Quat r; r.w = a.w; r.x = -a.x; r.y = -a.y; r.z = -a.z; return r; }
Quat qnormalize(Quat a) {
  double n = std::sqrt(a.w * a.w + a.x * a.x + a.y * a.y + a.z * a.z);
  Quat r; r.w = a.w / n; r.x = a.x / n; r.y = a.y / n; r.z = a.z / n;
  return r;
}

/* 3x3 rotation matrix of a unit quaternion. */
struct Mat3 {
  double m[3][3];
};
Mat3 rotation(Quat q) {
  Mat3 R;
  double w = q.w, x = q.x, y = q.y, z = q.z;
  R.m[0][0] = 1 - 2 * (y * y + z * z); R.m[0][1] = 2 * (x * y - w * z); R.m[0][2] = 2 * (x * z + w * y);
  R.m[1][0] = 2 * (x * y + w * z); R.m[1][1] = 1 - 2 * (x * x + z * z); R.m[1][2] = 2 * (y * z - w * x);
  R.m[2][0] = 2 * (x * z - w * y); R.m[2][1] = 2 * (y * z + w * x); R.m[2][2] = 1 - 2 * (x * x + y * y);
  return R;
}
Vec3 mul(const Mat3& R, Vec3 a) {
  return v3(R.m[0][0] * a.x + R.m[0][1] * a.y + R.m[0][2] * a.z,
            R.m[1][0] * a.x + R.m[1][1] * a.y + R.m[1][2] * a.z,
            R.m[2][0] * a.x + R.m[2][1] * a.y + R.m[2][2] * a.z);
}
Vec3 mulT(const Mat3& R, Vec3 a) {
  return v3(R.m[0][0] * a.x + R.m[1][0] * a.y + R.m[2][0] * a.z,
            R.m[0][1] * a.x + R.m[1][1] * a.y + R.m[2][1] * a.z,
            R.m[0][2] * a.x + R.m[1][2] * a.y + R.m[2][2] * a.z);
}

/* Pi: world -> bond frame for a bond along lattice axis (R5).
 * x-bond: identity; y-bond: (x,y,z)->(y,z,x); z-bond: (x,y,z)->(z,x,y). */
Vec3 perm_to_bond(int axis, Vec3 a) {
  if (axis == 0) return a;
  if (axis == 1) return v3(a.y, a.z, a.x);
  return v3(a.z, a.x, a.y);
}
/* Pi^-1: bond -> world frame. */
Vec3 perm_to_world(int axis, Vec3 a) {
  if (axis == 0) return a;
  if (axis == 1) return v3(a.z, a.x, a.y);
  return v3(a.y, a.z, a.x);
}

struct Material {
  double E, nu, rho, cte, mu_s, mu_d;
  double G;     /* G = E / (2(1+nu)) */
  double m, I;  /* m = rho l^3, I = m l^2 / 6 (R8) */
};

/* Composite and beam constants of a bond (Eq. 1-3, 4-12), plus damping. */
struct BondConst {
  double Ec, Gc, muc;
  double a1, a2, b1, b2, b3;
  double alpha_mean;  /* (alpha_1 + alpha_2)/2, Eq. 40 */
  double m_min, I_min;
};

struct Voxel {
  int i, j, k;
  int mat;         /* palette index (0-based) */
  bool fixed;
  Vec3 Fext;
  bool surface;
  int slot[6];     /* bond ids for -x,+x,-y,+y,-z,+z; -1 if none */
};

struct Bond {
  int a, b;        /* a on the negative side (R4) */
  int axis;        /* 0,1,2 */
  BondConst c;
};

struct StateV {
  Vec3 D;          /* position */
  Quat q;          /* orientation (theta, R6) */
  Vec3 P;          /* linear momentum */
  Vec3 phi;        /* angular momentum */
  bool latch;      /* static friction flag */
};

}  // namespace

struct orc_sim {
  int nx, ny, nz;
  double l;
  double origin[3];
  std::vector<Material> mats;
  orc_env env;
  std::vector<Voxel> vox;
  std::vector<Bond> bonds;
  std::vector<int> surface;   /* ascending voxel ids */
  std::vector<StateV> st;
  std::vector<int> cell_to_id;
  double dt;
  int64_t n;                   /* steps taken: t_n = n dt */
  int threads;
  std::vector<int> pending_region_kind;
};

namespace {

void composite(const Material& m1, const Material& m2, double& Ec, double& Gc, double& muc) {
  Ec = 2 * m1.E * m2.E / (m1.E + m2.E);   /* Eq. 1 */
  Gc = 2 * m1.G * m2.G / (m1.G + m2.G);   /* Eq. 2 */
  muc = Ec / (2 * Gc) - 1;                /* Eq. 3 */
}

void beam_constants(double Ec, double Gc, double l, double& a1, double& a2, double& b1,
                    double& b2, double& b3) {
  double A = l * l;
  double I = l * l * l * l / 12.0;   /* Eq. 4 */
  double J = l * l * l * l / 6.0;    /* Eq. 5 */
  a1 = Ec * A / l;                   /* Eq. 8 */
  a2 = Gc * J / l;                   /* Eq. 9 */
  b1 = 12 * Ec * I / (l * l * l);    /* Eq. 10 */
  b2 = 6 * Ec * I / (l * l);         /* Eq. 11 */
  b3 = 2 * Ec * I / l;               /* Eq. 12 */
}

BondConst make_bond_const(const Material& ma, const Material& mb, double l) {
  BondConst c;
  composite(ma, mb, c.Ec, c.Gc, c.muc);
  beam_constants(c.Ec, c.Gc, l, c.a1, c.a2, c.b1, c.b2, c.b3);
  c.alpha_mean = 0.5 * (ma.cte + mb.cte);
  c.m_min = std::min(ma.m, mb.m);
  c.I_min = std::min(ma.I, mb.I);
  return c;
}

/* Rest position of voxel (i,j,k): origin + l (i+1/2, j+1/2, k+1/2). */
Vec3 rest_position(const orc_sim* s, int i, int j, int k) {
  return v3(s->origin[0] + s->l * (i + 0.5), s->origin[1] + s->l * (j + 0.5),
            s->origin[2] + s->l * (k + 0.5));
}

double temperature_offset(const orc_sim* s, int64_t n) {
  /* T_n - T_r with T_n = T_r + A sin(2 pi f t_n + phase), t_n = n dt */
  double t = (double)n * s->dt;
  return s->env.T_amp * std::sin(2 * kPi * s->env.T_freq * t + s->env.T_phase);
}

/* One bond: world-frame loads on a (Fa, Ma) and b (Fb, Mb).
 * P:189 frame reduction; Eq. 13-24 (R1, R3); P:206 rotate back; Eq. 33-35. */
void bond_loads(const BondConst& c, int axis, double l, const StateV& A, const StateV& B,
                double mA, double IA, double mB, double IB, double zeta_bond, double dT,
                Vec3& Fa, Vec3& Ma, Vec3& Fb, Vec3& Mb) {
  /* Eq. 40: rest length at the current temperature. */
  double L_T = l * (1.0 + c.alpha_mean * dT);
  /* move voxel a to the origin with zero rotation, bond along +x. */
  Mat3 Ra = rotation(A.q);
  Vec3 r = B.D - A.D;
  Vec3 d = perm_to_bond(axis, mulT(Ra, r));
  Quat qrel = qmul(qconj(A.q), B.q);
  if (qrel.w < 0) { qrel.w = -qrel.w; qrel.x = -qrel.x; qrel.y = -qrel.y; qrel.z = -qrel.z; }
  Vec3 vq = v3(qrel.x, qrel.y, qrel.z);
  double vn = norm(vq);
  Vec3 th;
  if (vn > 0) th = (2.0 * std::atan2(vn, qrel.w) / vn) * vq;  /* R7 */
  th = perm_to_bond(axis, th);
  double X2 = d.x - L_T, Y2 = d.y, Z2 = d.z;
  double tx = th.x, ty = th.y, tz = th.z;
  /* Eq. 13-24, sign-fixed (R1) and negated (R3): loads on the voxels. */
  Vec3 fa = v3(c.a1 * X2, c.b1 * Y2 - c.b2 * tz, c.b1 * Z2 + c.b2 * ty);
  Vec3 ma = v3(c.a2 * tx, -c.b2 * Z2 - c.b3 * ty, c.b2 * Y2 - c.b3 * tz);
  Vec3 mb = v3(-c.a2 * tx, -c.b2 * Z2 - 2 * c.b3 * ty, c.b2 * Y2 - 2 * c.b3 * tz);
  /* transform back with the inverse of the frame transform. */
  Fa = mul(Ra, perm_to_world(axis, fa));
  Ma = mul(Ra, perm_to_world(axis, ma));
  Mb = mul(Ra, perm_to_world(axis, mb));
  /* Eq. 33-35: local bond damping (R10, R11), rigid motion removed. */
  if (zeta_bond > 0) {
    Vec3 VA = (1.0 / mA) * A.P, VB = (1.0 / mB) * B.P;
    Vec3 wA = (1.0 / IA) * A.phi, wB = (1.0 / IB) * B.phi;
    Vec3 Vavg = 0.5 * (VA + VB);
    Vec3 wavg = 0.5 * (wA + wB);
    Vec3 Vr = (VB - Vavg) + cross(0.5 * r, wavg);           /* Eq. 33 */
    double ct = 2 * zeta_bond * std::sqrt(c.m_min * c.a1);  /* Eq. 34 */
    Vec3 wr = wB - wavg;
    double cr = 2 * zeta_bond * std::sqrt(c.I_min * c.a2);  /* Eq. 35 */
    Fa = Fa + ct * Vr;     /* F_b gets -ct Vr, F_a gets +ct Vr */
    Ma = Ma + cr * wr;
    Mb = Mb - cr * wr;
  }
  Fb = -Fa;                /* Eq. 19-21 */
}

bool finite_state(const StateV& s) {
  double v[13] = {s.D.x, s.D.y, s.D.z, s.q.w, s.q.x, s.q.y, s.q.z,
                  s.P.x, s.P.y, s.P.z, s.phi.x, s.phi.y, s.phi.z};
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

int manhattan(const Voxel& a, const Voxel& b) {
  return std::abs(a.i - b.i) + std::abs(a.j - b.j) + std::abs(a.k - b.k);
}

/* Contact force on voxel a from voxel b (row a7 / R16). */
Vec3 contact_force(const orc_sim* s, int a, int b, double dT) {
  const Voxel& va = s->vox[a];
  const Voxel& vb = s->vox[b];
  const Material& ma = s->mats[va.mat];
  const Material& mb = s->mats[vb.mat];
  double ra = 0.5 * s->l * (1.0 + ma.cte * dT);
  double rb = 0.5 * s->l * (1.0 + mb.cte * dT);
  Vec3 d = s->st[a].D - s->st[b].D;
  double dist = norm(d);
  double q = ra + rb - dist;
  if (!(q > 0)) return Vec3();
  Vec3 n;
  /* coincident centres (reading R16: closer than 1e-6 l, where the
   * centre line is rounding noise in any stored representation): +z for the
   * lower id, -z for the other */
  if (dist > 1e-6 * s->l) n = (1.0 / dist) * d;
  else n = v3(0, 0, a < b ? 1.0 : -1.0);
  Vec3 Va = (1.0 / ma.m) * s->st[a].P, Vb = (1.0 / mb.m) * s->st[b].P;
  double vnrm = dot(Va - Vb, n);
  double ka = ma.E * s->l, kb = mb.E * s->l;
  double kc = 2 * ka * kb / (ka + kb);
  double cc = 2 * s->env.zeta_col * std::sqrt(std::min(ma.m, mb.m) * kc);
  double f = kc * q - cc * vnrm;
  if (f < 0) f = 0;
  return f * n;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void orc_composite(double E1, double nu1, double E2, double nu2, double out[3]) {
  Material a{}, b{};
  a.E = E1; a.nu = nu1; a.G = E1 / (2 * (1 + nu1));
  b.E = E2; b.nu = nu2; b.G = E2 / (2 * (1 + nu2));
  composite(a, b, out[0], out[1], out[2]);
}

void orc_beam_constants(double Ec, double Gc, double l, double out[5]) {
  beam_constants(Ec, Gc, l, out[0], out[1], out[2], out[3], out[4]);
}

orc_sim* orc_create(int32_t nx, int32_t ny, int32_t nz, double l, const double origin[3],
                    const uint8_t* cells, const orc_material* mats, int32_t nmat,
                    const orc_env* env) {
  if (nx < 0 || ny < 0 || nz < 0 || !(l > 0) || !cells || !env || nmat < 1 || nmat > 255) {
    g_err = "invalid lattice";
    return nullptr;
  }
  orc_sim* s = new orc_sim();
  s->nx = nx; s->ny = ny; s->nz = nz; s->l = l;
  for (int d = 0; d < 3; ++d) s->origin[d] = origin ? origin[d] : 0.0;
  s->env = *env;
  s->n = 0;
  s->threads = 1;
  for (int m = 0; m < nmat; ++m) {
    Material M;
    M.E = mats[m].E; M.nu = mats[m].nu; M.rho = mats[m].rho; M.cte = mats[m].cte;
    M.mu_s = mats[m].mu_s; M.mu_d = mats[m].mu_d;
    if (!(M.E > 0) || !(M.rho > 0) || !(M.nu > -1 && M.nu < 0.5) || !(M.mu_d >= 0) ||
        !(M.mu_s >= M.mu_d)) {
      g_err = "invalid material " + std::to_string(m);
      delete s;
      return nullptr;
    }
    M.G = M.E / (2 * (1 + M.nu));
    M.m = M.rho * l * l * l;
    M.I = M.m * l * l / 6.0;
    s->mats.push_back(M);
  }
  /* voxels: filled cells in x-fastest order */
  size_t ncell = (size_t)nx * ny * nz;
  s->cell_to_id.assign(ncell, -1);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        size_t c = (size_t)i + (size_t)nx * (j + (size_t)ny * k);
        if (cells[c] == 0) continue;
        if (cells[c] > nmat) {
          g_err = "cell material index out of range";
          delete s;
          return nullptr;
        }
        Voxel v;
        v.i = i; v.j = j; v.k = k; v.mat = cells[c] - 1;
        v.fixed = false; v.surface = false;
        for (int q = 0; q < 6; ++q) v.slot[q] = -1;
        s->cell_to_id[c] = (int)s->vox.size();
        s->vox.push_back(v);
      }
  auto id_at = [&](int i, int j, int k) -> int {
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return -1;
    return s->cell_to_id[(size_t)i + (size_t)nx * (j + (size_t)ny * k)];
  };
  /* bonds between face neighbours, a on the negative side (R4) */
  for (size_t a = 0; a < s->vox.size(); ++a) {
    Voxel& va = s->vox[a];
    int nbr[3] = {id_at(va.i + 1, va.j, va.k), id_at(va.i, va.j + 1, va.k),
                  id_at(va.i, va.j, va.k + 1)};
    for (int ax = 0; ax < 3; ++ax) {
      int b = nbr[ax];
      if (b < 0) continue;
      Bond B;
      B.a = (int)a; B.b = b; B.axis = ax;
      B.c = make_bond_const(s->mats[va.mat], s->mats[s->vox[b].mat], l);
      int id = (int)s->bonds.size();
      s->bonds.push_back(B);
      s->vox[a].slot[2 * ax + 1] = id;  /* +axis slot of a */
      s->vox[b].slot[2 * ax] = id;      /* -axis slot of b */
    }
  }
  /* surface voxels: fewer than 6 filled neighbours */
  for (size_t v = 0; v < s->vox.size(); ++v) {
    int cnt = 0;
    for (int q = 0; q < 6; ++q) cnt += s->vox[v].slot[q] >= 0;
    s->vox[v].surface = cnt < 6;
    if (cnt < 6) s->surface.push_back((int)v);
  }
  /* Eq. 31-32 (R9): omega_0m = max over bonds of sqrt(k_b / m_min). */
  double w2max = 0;
  for (const Bond& B : s->bonds) w2max = std::max(w2max, B.c.a1 / B.c.m_min);
  if (s->bonds.empty())
    for (const Voxel& v : s->vox) {
      const Material& M = s->mats[v.mat];
      w2max = std::max(w2max, M.E * l / M.m);
    }
  s->dt = w2max > 0 ? env->dt_safety / (2 * kPi * std::sqrt(w2max)) : 0.0;
  /* initial state: at rest on the lattice sites */
  s->st.resize(s->vox.size());
  for (size_t v = 0; v < s->vox.size(); ++v) {
    StateV& x = s->st[v];
    x.D = rest_position(s, s->vox[v].i, s->vox[v].j, s->vox[v].k);
    x.latch = false;
  }
  return s;
}

void orc_destroy(orc_sim* s) { delete s; }

int64_t orc_num_voxels(const orc_sim* s) { return (int64_t)s->vox.size(); }
int64_t orc_num_bonds(const orc_sim* s) { return (int64_t)s->bonds.size(); }
int64_t orc_num_surface(const orc_sim* s) { return (int64_t)s->surface.size(); }
double orc_dt(const orc_sim* s) { return s->dt; }

int orc_set_boundary(orc_sim* s, const uint8_t* fixed, const double* fext) {
  for (size_t v = 0; v < s->vox.size(); ++v) {
    s->vox[v].fixed = fixed ? fixed[v] != 0 : false;
    s->vox[v].Fext = fext ? v3(fext[3 * v], fext[3 * v + 1], fext[3 * v + 2]) : Vec3();
  }
  return 0;
}

/* App. B: a voxel belongs to the region if its cell box
 * intersects the region box (positive overlap on every axis, or, for a
 * zero-width region axis, the plane lies within the closed cell interval).
 * Fixed takes precedence; a forced region's force is split equally over
 * every filled voxel it touches. */
int orc_add_region(orc_sim* s, int32_t kind, const double o[3], const double sz[3],
                   const double force[3]) {
  int dims[3] = {s->nx, s->ny, s->nz};
  std::vector<int> hit;
  for (size_t v = 0; v < s->vox.size(); ++v) {
    int idx[3] = {s->vox[v].i, s->vox[v].j, s->vox[v].k};
    bool in = true;
    for (int d = 0; d < 3; ++d) {
      double lo = o[d] * dims[d], hi = (o[d] + sz[d]) * dims[d];  /* in cell units */
      double c0 = idx[d], c1 = idx[d] + 1.0;
      bool overlap = (hi > lo) ? (std::max(lo, c0) < std::min(hi, c1)) : (c0 <= lo && lo <= c1);
      if (!overlap) { in = false; break; }
    }
    if (in) hit.push_back((int)v);
  }
  if (kind == 0) {
    for (int v : hit) s->vox[v].fixed = true;
  } else if (kind == 1) {
    if (hit.empty()) return 0;
    double inv = 1.0 / (double)hit.size();
    Vec3 f = v3(force[0] * inv, force[1] * inv, force[2] * inv);
    for (int v : hit) s->vox[v].Fext = s->vox[v].Fext + f;
  } else {
    g_err = "bad region kind";
    return -1;
  }
  return 0;
}

int orc_set_state(orc_sim* s, const double* pos, const double* quat, const double* linmom,
                  const double* angmom, const uint8_t* latch) {
  for (size_t v = 0; v < s->vox.size(); ++v) {
    StateV& x = s->st[v];
    if (pos) x.D = v3(pos[3 * v], pos[3 * v + 1], pos[3 * v + 2]);
    if (quat) { x.q.w = quat[4 * v]; x.q.x = quat[4 * v + 1]; x.q.y = quat[4 * v + 2]; x.q.z = quat[4 * v + 3]; }
    if (linmom) x.P = v3(linmom[3 * v], linmom[3 * v + 1], linmom[3 * v + 2]);
    if (angmom) x.phi = v3(angmom[3 * v], angmom[3 * v + 1], angmom[3 * v + 2]);
    if (latch) x.latch = latch[v] != 0;
  }
  return 0;
}

int orc_read_state(const orc_sim* s, double* pos, double* quat, double* linmom, double* angmom,
                   uint8_t* latch) {
  for (size_t v = 0; v < s->vox.size(); ++v) {
    const StateV& x = s->st[v];
    if (pos) { pos[3 * v] = x.D.x; pos[3 * v + 1] = x.D.y; pos[3 * v + 2] = x.D.z; }
    if (quat) { quat[4 * v] = x.q.w; quat[4 * v + 1] = x.q.x; quat[4 * v + 2] = x.q.y; quat[4 * v + 3] = x.q.z; }
    if (linmom) { linmom[3 * v] = x.P.x; linmom[3 * v + 1] = x.P.y; linmom[3 * v + 2] = x.P.z; }
    if (angmom) { angmom[3 * v] = x.phi.x; angmom[3 * v + 1] = x.phi.y; angmom[3 * v + 2] = x.phi.z; }
    if (latch) latch[v] = x.latch ? 1 : 0;
  }
  return 0;
}

int orc_set_step(orc_sim* s, int64_t n) { s->n = n; return 0; }
int64_t orc_get_step(const orc_sim* s) { return s->n; }
int orc_set_threads(orc_sim* s, int32_t n) { s->threads = n < 1 ? 1 : n; return 0; }
int orc_set_dt(orc_sim* s, double dt) { s->dt = dt; return 0; }

void orc_bond_loads(const orc_sim* s, int32_t a_mat, int32_t b_mat, int32_t axis,
                    const double* sa, const double* sb, double dT, double out[12]) {
  const Material& ma = s->mats[a_mat];
  const Material& mb = s->mats[b_mat];
  BondConst c = make_bond_const(ma, mb, s->l);
  StateV A, B;
  A.D = v3(sa[0], sa[1], sa[2]); A.q.w = sa[3]; A.q.x = sa[4]; A.q.y = sa[5]; A.q.z = sa[6];
  A.P = v3(sa[7], sa[8], sa[9]); A.phi = v3(sa[10], sa[11], sa[12]);
  B.D = v3(sb[0], sb[1], sb[2]); B.q.w = sb[3]; B.q.x = sb[4]; B.q.y = sb[5]; B.q.z = sb[6];
  B.P = v3(sb[7], sb[8], sb[9]); B.phi = v3(sb[10], sb[11], sb[12]);
  Vec3 Fa, Ma, Fb, Mb;
  bond_loads(c, axis, s->l, A, B, ma.m, ma.I, mb.m, mb.I, s->env.zeta_bond, dT, Fa, Ma, Fb, Mb);
  double o[12] = {Fa.x, Fa.y, Fa.z, Ma.x, Ma.y, Ma.z, Fb.x, Fb.y, Fb.z, Mb.x, Mb.y, Mb.z};
  std::memcpy(out, o, sizeof o);
}

int64_t orc_contact_pairs(const orc_sim* s, int32_t* pairs, int64_t cap) {
  double dT = temperature_offset(s, s->n);
  int64_t cnt = 0;
  for (size_t x = 0; x < s->surface.size(); ++x)
    for (size_t y = x + 1; y < s->surface.size(); ++y) {
      int a = s->surface[x], b = s->surface[y];
      if (manhattan(s->vox[a], s->vox[b]) <= 3) continue;
      const Material& ma = s->mats[s->vox[a].mat];
      const Material& mb = s->mats[s->vox[b].mat];
      double ra = 0.5 * s->l * (1.0 + ma.cte * dT), rb = 0.5 * s->l * (1.0 + mb.cte * dT);
      double dist = norm(s->st[a].D - s->st[b].D);
      if (ra + rb - dist > 0) {
        if (cnt < cap) { pairs[2 * cnt] = a; pairs[2 * cnt + 1] = b; }
        ++cnt;
      }
    }
  return cnt;
}

/* One synchronous step n -> n+1: all loads from the frozen state,
 * then all voxels updated (Eq. 27-30). */
static int step_once(orc_sim* s) {
  const double dt = s->dt;
  const double l = s->l;
  const orc_env& env = s->env;
  const double dT = temperature_offset(s, s->n);
  const int64_t NB = (int64_t)s->bonds.size();
  const int64_t NV = (int64_t)s->vox.size();

  /* Eq. 40: a non-positive rest length is a fault. */
  for (const Bond& B : s->bonds)
    if (!(l * (1.0 + B.c.alpha_mean * dT) > 0)) {
      g_err = "non-positive thermal rest length at step " + std::to_string(s->n);
      return -6;
    }

  /* phase 1a: every bond's loads from the frozen state */
  std::vector<Vec3> Fa(NB), Ma(NB), Fb(NB), Mb(NB);
#pragma omp parallel for num_threads(s->threads) schedule(static)
  for (int64_t b = 0; b < NB; ++b) {
    const Bond& B = s->bonds[b];
    const Material& ma = s->mats[s->vox[B.a].mat];
    const Material& mb = s->mats[s->vox[B.b].mat];
    bond_loads(B.c, B.axis, l, s->st[B.a], s->st[B.b], ma.m, ma.I, mb.m, mb.I, env.zeta_bond,
               dT, Fa[b], Ma[b], Fb[b], Mb[b]);
  }

  /* phase 1b + 2: per voxel sums (Eq. 25-26), environment, integration */
  std::vector<StateV> next(s->st);
#pragma omp parallel for num_threads(s->threads) schedule(static)
  for (int64_t v = 0; v < NV; ++v) {
    const Voxel& vx = s->vox[v];
    if (vx.fixed) continue;             /* fixed voxels are kinematic */
    const Material& M = s->mats[vx.mat];
    const StateV& x = s->st[v];
    const Vec3 V = (1.0 / M.m) * x.P;   /* velocity */
    const Vec3 w = (1.0 / M.I) * x.phi; /* angular velocity (world, isotropic I) */
    Vec3 F, Mt;
    /* slots -x,+x,-y,+y,-z,+z: a -axis slot holds the bond (v-e, v), v is "b" */
    for (int q = 0; q < 6; ++q) {
      int b = vx.slot[q];
      if (b < 0) continue;
      if (q % 2 == 0) { F = F + Fb[b]; Mt = Mt + Mb[b]; }
      else { F = F + Fa[b]; Mt = Mt + Ma[b]; }
    }
    F = F + vx.Fext;                                  /* forced regions */
    F.z = F.z - M.m * env.gravity;
    if (env.zeta_ground > 0) {                        /* P:254, R12 */
      double cgt = 2 * env.zeta_ground * std::sqrt(M.m * M.E * l);
      double cgr = 2 * env.zeta_ground * std::sqrt(M.I * M.G * l * l * l / 6.0);
      F = F - cgt * V;
      Mt = Mt - cgr * w;
    }
    if (env.self_collision && vx.surface) {           /* P:276-282, R16 */
      for (int p : s->surface) {
        if (p == v) continue;
        if (manhattan(vx, s->vox[p]) <= 3) continue;
        F = F + contact_force(s, (int)v, p, dT);
      }
    }
    bool latch = x.latch;
    bool zero_lat = false;
    if (env.floor_on) {                               /* P:260-274, R14, R15 */
      double rv = 0.5 * l * (1.0 + M.cte * dT);
      double pen = rv - (x.D.z - env.floor_z);
      if (pen > 0) {
        double kf = M.E * l;
        double cf = 2 * env.zeta_col * std::sqrt(M.m * kf);
        double Fn = kf * pen - cf * V.z;
        if (Fn < 0) Fn = 0;
        F.z = F.z + Fn;
        double Flx = F.x, Fly = F.y;
        double Fl = std::sqrt(Flx * Flx + Fly * Fly);
        double Vl = std::sqrt(V.x * V.x + V.y * V.y);
        if (latch) {
          if (Fl <= M.mu_s * Fn) {                    /* Eq. 36 not exceeded */
            F.x = 0; F.y = 0; zero_lat = true;
          } else {                                    /* break away: Eq. 37 */
            latch = false;
            F.x = Flx - M.mu_d * Fn * Flx / Fl;
            F.y = Fly - M.mu_d * Fn * Fly / Fl;
          }
        } else {
          if (Vl <= M.mu_d * Fn * dt / M.m) {         /* Eq. 38: halt */
            F.x = 0; F.y = 0; zero_lat = true; latch = true;
          } else {                                    /* Eq. 37 opposing motion */
            F.x = Flx - M.mu_d * Fn * V.x / Vl;
            F.y = Fly - M.mu_d * Fn * V.y / Vl;
          }
        }
      } else {
        latch = false;
      }
    }
    /* Eq. 27-30 (R6) */
    StateV& y = next[v];
    y.P = x.P + dt * F;                               /* Eq. 27 */
    if (zero_lat) { y.P.x = 0; y.P.y = 0; }
    y.D = x.D + (dt / M.m) * y.P;                     /* Eq. 28 */
    y.phi = x.phi + dt * Mt;                          /* Eq. 29 */
    Vec3 th = (dt / M.I) * y.phi;                     /* Eq. 30 increment */
    double a = norm(th);
    Quat dq;
    if (a > 0) {
      double sa = std::sin(0.5 * a) / a;
      dq.w = std::cos(0.5 * a); dq.x = sa * th.x; dq.y = sa * th.y; dq.z = sa * th.z;
    }
    y.q = qnormalize(qmul(dq, x.q));
    y.latch = latch;
  }
  s->st.swap(next);
  for (int64_t v = 0; v < NV; ++v)
    if (!finite_state(s->st[v])) {
      g_err = "diverged: voxel " + std::to_string(v) + " at step " + std::to_string(s->n);
      s->n += 1;
      return -6;
    }
  s->n += 1;
  return 0;
}

int orc_step(orc_sim* s, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    int r = step_once(s);
    if (r) return r;
  }
  return 0;
}

}  // extern "C"
