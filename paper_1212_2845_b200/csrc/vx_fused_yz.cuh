// vx_fused_yz.cuh -- the fused step for shallow lattices (nz < 64).
//
// k_step_fused maps one thread to each z and runs a tile's rows one after the
// other, so a lattice with nz = 16 leaves half of every warp idle and its rows
// form a long serial chain.  Here a block holds G = floor(256 / nz) rows side
// by side (thread t -> row r = t / nz of the group, layer k = t % nz) and sweeps
// a tile of TY = G x M rows in M steps.  Per voxel the work is k_step_fused's:
// the same bond_eval calls, the same slot order (-x, +x, -y, +y, -z, +z) and
// finish_voxel, so S_{n+1} is bitwise the same.  What changes is where the -y
// record comes from: the +y bond of row j - 1 is evaluated in the same step by
// the group below (r > 0), or by group G - 1 one step earlier (r = 0), or as
// the tile's halo row j0 - 1 at the start of a plane; it goes through a
// three-slot shared ring, so the -y slot is added after the step's barrier
// (the sum order is unchanged: -x and +x are summed before it).
#pragma once
#include "vx_kernels.cuh"

namespace vx {

template <class R> size_t fused_yz_smem(int ty, int nz, int g) {
  // xrec[ty][nz], yring[3][g * nz], zrec[2][g * nz] (+ their row tags, checked build)
  return sizeof(Rec6<R>) * ((size_t)ty * nz + 5 * (size_t)g * nz)
#ifdef VX_CHECKED
         + sizeof(int) * 5 * (size_t)g * nz
#endif
      ;
}

template <class R, bool COLLIDE>
__global__ void __launch_bounds__(256, sizeof(R) == 4 ? 2 : 1) k_step_fused_yz(Dev<R> d, FusedArgs<R> a) {
  using R4 = typename VT<R>::R4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nz = (int)d.nz, G = a.zchunks;   // zchunks carries G (rows side by side)
  const int gn = G * nz;
  Rec6<R>* xrec = reinterpret_cast<Rec6<R>*>(smem_raw);
  Rec6<R>* yring = xrec + (size_t)a.ty * nz;
  Rec6<R>* zrec = yring + 3 * (size_t)gn;
  const int t = threadIdx.x, r = t / nz, k = t - r * nz;
  const bool lane_ok = t < gn;
#ifdef VX_CHECKED
  volatile int* rtag = reinterpret_cast<volatile int*>(zrec + 2 * (size_t)gn);   // [3][gn]
  volatile int* ztag = rtag + 3 * gn;                                             // [2][gn]
  for (int q = t; q < 5 * gn; q += blockDim.x) rtag[q] = -1;
  __syncthreads();
#endif

  int bid = blockIdx.x, p0 = a.p0, p1 = a.p1;
  if (bid >= a.nblk0) { bid -= a.nblk0; p0 = a.p0b; p1 = a.p1b; }
  const int tile = bid % a.ntiles_y;
  const int seg = bid / a.ntiles_y;
  const int j0 = tile * a.ty;
  const int j1 = min(j0 + a.ty, (int)d.ny);
  const int i0 = p0 + seg * a.sx;
  const int i1 = min(i0 + a.sx, p1);
  const uint32_t sx = d.sx;
  const R dT = (R)d.clk->dT;
  const R kf = floor_base(d, (uint32_t)k);
  R vmax = R(0);
  auto idx = [&](int i, int j) { return (uint32_t)i * sx + (uint32_t)j * (uint32_t)nz + (uint32_t)k; };
  const int steps = (j1 - j0 + G - 1) / G;
  auto slot = [&](int m) { return yring + (size_t)((m + 3) % 3) * gn; };   // ring slot of step m >= -1
  int pl = 0;   // planes done (row tags: stamp of step m of this plane)
  auto stamp = [&](int m) { return pl * (steps + 1) + m + 1; };
  (void)stamp;

  // -x slots of plane i0: the +x bonds of plane i0 - 1 (halo, recomputed)
  for (int m = 0; m < steps; ++m) {
    const int j = j0 + m * G + r;
    if (!lane_ok || j >= j1) continue;
    Rec6<R> rx{};
    if (i0 > 0) {
      const VS<R> va = ldv(d, idx(i0 - 1, j));
      const VS<R> vb = ldv(d, idx(i0, j));
      if (meta_of(va.p.w) & nb_bit(1)) {
        const AFrame<R> f = a_frame(d, va);
        V3<R> Fa, Ma, Mb;
        bond_eval<0>(d, f.Ra, va.q, f.ua, f.Va, f.wa, f.mat, vb, dT, Fa, Ma, Mb);
        rx = rec6(Fa, Mb);
      }
    }
    xrec[(size_t)(j - j0) * nz + k] = rx;
  }

  for (int i = i0; i < i1; ++i) {
    __syncthreads();   // the previous plane's ring reads are done
    // halo row j0 - 1: its +y bond, in the slot group G - 1 fills at step -1
    if (lane_ok && r == G - 1) {
      Rec6<R> ry{};
      if (j0 > 0) {
        const VS<R> vh = ldv(d, idx(i, j0 - 1));
        if (meta_of(vh.p.w) & nb_bit(3)) {
          const VS<R> vb = ldv(d, idx(i, j0));
          const AFrame<R> f = a_frame(d, vh);
          V3<R> Fa, Ma, Mb;
          bond_eval<1>(d, f.Ra, vh.q, f.ua, f.Va, f.wa, f.mat, vb, dT, Fa, Ma, Mb);
          ry = rec6(Fa, Mb);
        }
      }
      slot(-1)[t] = ry;
      VX_CHECKED_ONLY(__threadfence_block(); rtag[2 * gn + t] = stamp(-1));
    }
    for (int m = 0; m < steps; ++m) {
      const int j = j0 + m * G + r;
      const bool act = lane_ok && j < j1;
      const uint32_t id = act ? idx(i, j) : 0u;
      VS<R> cur{};
      if (act) cur = ldv(d, id);
      const uint32_t meta = act ? meta_of(cur.p.w) : 0u;
      VS<R> vy{}, vx{};
      if (meta & nb_bit(3)) vy = ldv(d, id + (uint32_t)nz);
      if (meta & nb_bit(1)) vx = ldv(d, id + sx);
      if (act && i + 1 < a.nplanes) {   // the next step's +x rows (first touch: HBM) into L2
        int jj = j + G, ii = i + 1;
        if (jj >= j1) { jj -= j1 - j0; ++ii; }
        if (ii < a.nplanes && (ii == i + 1 || i + 1 < i1)) {
          const uint32_t f = idx(ii, jj);
          prefetch_l2(d.pos + f);
          prefetch_l2(d.quat + f);
          prefetch_l2(d.mom + f);
          prefetch_l2(d.ang + f);
        }
      }
      // +z neighbour: the next thread's voxel (same row when k + 1 < nz); the
      // last lane of a warp reads it
      VS<R> vz = vs_shfl_down(cur);
      if ((t & 31) == 31 && (meta & nb_bit(5))) vz = ldv(d, id + 1);
      V3<R> FX{}, MX{}, BX{}, FY{}, MY{}, BY{}, FZ{}, MZ{}, BZ{};
      if (meta & M_FILLED) {
        const AFrame<R> f = a_frame(d, cur);
        if (meta & nb_bit(5)) bond_eval<2>(d, f.Ra, cur.q, f.ua, f.Va, f.wa, f.mat, vz, dT, FZ, MZ, BZ);
        if (meta & nb_bit(1)) bond_eval<0>(d, f.Ra, cur.q, f.ua, f.Va, f.wa, f.mat, vx, dT, FX, MX, BX);
        if (meta & nb_bit(3)) bond_eval<1>(d, f.Ra, cur.q, f.ua, f.Va, f.wa, f.mat, vy, dT, FY, MY, BY);
      }
      Rec6<R>* zr = zrec + (size_t)(m & 1) * gn;
      if (lane_ok) {
        zr[t] = rec6(FZ, BZ);
        slot(m)[t] = rec6(FY, BY);
        VX_CHECKED_ONLY(__threadfence_block(); ztag[(m & 1) * gn + t] = stamp(m);
                        rtag[((m + 3) % 3) * gn + t] = stamp(m));
      }
      V3<R> F = mk(R(0), R(0), R(0)), M = F;
      if (act) {
        Rec6<R>& xr = xrec[(size_t)(j - j0) * nz + k];
        if (meta & nb_bit(0)) slot_minus(F, M, xr);
        if (meta & nb_bit(1)) slot_plus(F, M, FX, MX);
        if (meta & M_FILLED) xr = rec6(FX, BX);
      }
      __syncthreads();
      if (!act) continue;
      VX_CHK(i >= p0 && i < p1, 7);
      if ((meta & (M_FILLED | M_FIXED)) == M_FILLED) {
#ifdef VX_CHECKED
        if ((t & 31) == 0) __nanosleep(((unsigned)(t * 613 + m * 97 + pl * 31)) % 2000u);
        if (meta & nb_bit(2))
          VX_CHK(r > 0 ? rtag[((m + 3) % 3) * gn + t - nz] == stamp(m)
                       : rtag[((m + 2) % 3) * gn + t + (G - 1) * nz] == stamp(m - 1), 5);
        if (meta & nb_bit(4)) VX_CHK(ztag[(m & 1) * gn + t - 1] == stamp(m), 6);
#endif
        if (meta & nb_bit(2)) slot_minus(F, M, r > 0 ? slot(m)[t - nz] : slot(m - 1)[t + (G - 1) * nz]);
        if (meta & nb_bit(3)) slot_plus(F, M, FY, MY);
        if (meta & nb_bit(4)) slot_minus(F, M, zr[t - 1]);
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
    }
    ++pl;
  }
  if constexpr (COLLIDE) budget_max(d, vmax);
}

}  // namespace vx
