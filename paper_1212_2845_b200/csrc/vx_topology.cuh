// vx_topology.cuh -- K1: the lattice build on the device.
//
// From the input grid (uint8 per cell, x-fastest, 0 = empty, k = material k-1):
//   external ids   filled cells in x-fastest order: a scan of the filled flags
//                  gives each cell its external id, a scatter the box id of each
//                  external id (box order: x slowest, z fastest);
//   static meta    per local box voxel: material, FILLED, the six neighbour bits
//                  (-x,+x,-y,+y,-z,+z) and SURF (< 6 neighbours);
//   counts         bonds (a voxel's +x/+y/+z neighbours), surface voxels, the
//                  largest material index, and the material pairs present on
//                  bonds (a on the negative side) as a 256 x 256 bit table;
//   surface list   global box ids of the surface voxels in ascending order
//                  (a scan of the surface flags in box order).
// Boundary conditions go the same way: fixed flags and external forces of the
// external voxels are scattered into the local boxes (k_apply_bc).
#pragma once
#include "vx_common.cuh"

namespace vx {

__device__ __forceinline__ int topo_cell(const uint8_t* cells, int nx, int ny, int nz, int i, int j,
                                         int k) {
  if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return 0;
  return cells[(size_t)i + (size_t)nx * ((size_t)j + (size_t)ny * (size_t)k)];
}

// Static meta of filled cell (i, j, k) with material index c >= 1.
__device__ __forceinline__ uint32_t topo_meta(const uint8_t* cells, int nx, int ny, int nz, int i,
                                              int j, int k, int c) {
  const int di[6] = {-1, 1, 0, 0, 0, 0}, dj[6] = {0, 0, -1, 1, 0, 0}, dk[6] = {0, 0, 0, 0, -1, 1};
  uint32_t m = (uint32_t)(c - 1) | M_FILLED;
  int cnt = 0;
#pragma unroll
  for (int s = 0; s < 6; ++s)
    if (topo_cell(cells, nx, ny, nz, i + di[s], j + dj[s], k + dk[s])) {
      m |= nb_bit(s);
      ++cnt;
    }
  if (cnt < 6) m |= M_SURF;
  return m;
}

// filled flag per cell, x-fastest order
__global__ void k_topo_filled(const uint8_t* cells, unsigned long long n, uint32_t* flag) {
  for (unsigned long long f = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; f < n;
       f += (unsigned long long)gridDim.x * blockDim.x)
    flag[f] = cells[f] ? 1u : 0u;
}

// box id of every external id (ext = exclusive scan of the filled flags)
__global__ void k_topo_ext(const uint8_t* cells, int nx, int ny, int nz, unsigned long long n,
                           const uint32_t* ext, long long* box_of_ext) {
  for (unsigned long long f = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; f < n;
       f += (unsigned long long)gridDim.x * blockDim.x) {
    if (!cells[f]) continue;
    const long long i = (long long)(f % (unsigned long long)nx);
    const long long j = (long long)((f / (unsigned long long)nx) % (unsigned long long)ny);
    const long long k = (long long)(f / ((unsigned long long)nx * ny));
    box_of_ext[ext[f]] = (i * ny + j) * nz + k;
  }
}

// Counts, pair table and surface flags over every box id.
// counts[0] bonds, counts[1] surface voxels; pair_bits: 2048 words.
__global__ void __launch_bounds__(256) k_topo_count(const uint8_t* cells, int nx, int ny, int nz,
                                                    unsigned long long nbox,
                                                    unsigned long long* counts, unsigned* pair_bits,
                                                    int* max_cell, uint32_t* surf_flag) {
  __shared__ unsigned sp[2048];
  __shared__ unsigned long long red[2][8];
  __shared__ int redm[8];
  for (int x = threadIdx.x; x < 2048; x += blockDim.x) sp[x] = 0;
  __syncthreads();
  unsigned long long nb = 0, ns = 0;
  int mc = 0;
  const unsigned long long plane = (unsigned long long)ny * nz;
  for (unsigned long long b = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; b < nbox;
       b += (unsigned long long)gridDim.x * blockDim.x) {
    const int i = (int)(b / plane);
    const unsigned long long r = b - (unsigned long long)i * plane;
    const int j = (int)(r / nz), k = (int)(r - (unsigned long long)j * nz);
    const int c = topo_cell(cells, nx, ny, nz, i, j, k);
    uint32_t sf = 0;
    if (c) {
      mc = max(mc, c);
      const uint32_t m = topo_meta(cells, nx, ny, nz, i, j, k, c);
      const int pi[3] = {1, 0, 0}, pj[3] = {0, 1, 0}, pk[3] = {0, 0, 1};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (!(m & nb_bit(2 * a + 1))) continue;
        ++nb;
        const int cb = topo_cell(cells, nx, ny, nz, i + pi[a], j + pj[a], k + pk[a]);
        const unsigned idx = (unsigned)(c - 1) * 256u + (unsigned)(cb - 1);
        const unsigned bit = 1u << (idx & 31u);
        if (!(sp[idx >> 5] & bit)) atomicOr(&sp[idx >> 5], bit);
      }
      if (m & M_SURF) {
        ++ns;
        sf = 1;
      }
    }
    surf_flag[b] = sf;
  }
  // block reductions
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
    ns += __shfl_xor_sync(0xffffffffu, ns, o);
    mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = nb;
    red[1][warp] = ns;
    redm[warp] = mc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0, s = 0;
    int m = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += red[0][w];
      s += red[1][w];
      m = max(m, redm[w]);
    }
    if (a) atomicAdd(&counts[0], a);
    if (s) atomicAdd(&counts[1], s);
    if (m) atomicMax(max_cell, m);
  }
  for (int x = threadIdx.x; x < 2048; x += blockDim.x)
    if (sp[x]) atomicOr(&pair_bits[x], sp[x]);
}

// surface list: global box ids of the surface voxels, ascending (sidx = scan of the flags)
__global__ void k_topo_surf(const uint32_t* surf_flag, const uint32_t* sidx, unsigned long long nbox,
                            unsigned* surf_g) {
  for (unsigned long long b = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; b < nbox;
       b += (unsigned long long)gridDim.x * blockDim.x)
    if (surf_flag[b]) surf_g[sidx[b]] = (unsigned)b;
}

// static meta of one slab's local box (global planes [xl0, xl0 + nloc / plane))
__global__ void k_topo_meta(const uint8_t* cells, int nx, int ny, int nz, int xl0, uint32_t nloc,
                            uint32_t* meta) {
  const uint32_t li = blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= nloc) return;
  const uint32_t plane = (uint32_t)ny * (uint32_t)nz;
  const int i = xl0 + (int)(li / plane);
  const uint32_t r = li % plane;
  const int j = (int)(r / (uint32_t)nz), k = (int)(r % (uint32_t)nz);
  const int c = topo_cell(cells, nx, ny, nz, i, j, k);
  meta[li] = c ? topo_meta(cells, nx, ny, nz, i, j, k, c) : 0u;
}

// external id of every local box voxel (0xffffffff: empty cell)
__global__ void k_topo_eol(const long long* box_of_ext, long long n, long long box_base, uint32_t nloc,
                           uint32_t* ext_of_local) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long li = box_of_ext[e] - box_base;
    if (li >= 0 && li < (long long)nloc) ext_of_local[li] = (uint32_t)e;
  }
}

// identity orientation
template <class R> __global__ void k_topo_quat_identity(typename VT<R>::R4* q, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) q[i] = typename VT<R>::R4{R(0), R(0), R(0), R(1)};
}

// boundary conditions of the external voxels into one slab's meta (FIXED, EXT)
// and external-force array (zero elsewhere)
template <class R>
__global__ void k_apply_bc(const long long* box_of_ext, long long n, long long box_base, uint32_t nloc,
                           const uint8_t* fixed, const double* fext, uint32_t* meta,
                           typename VT<R>::R4* fextd) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long li = box_of_ext[e] - box_base;
    if (li < 0 || li >= (long long)nloc) continue;
    uint32_t m = meta[li] & ~(M_FIXED | M_EXT);
    if (fixed && fixed[e]) m |= M_FIXED;
    if (fext) {
      const double fx = fext[3 * e], fy = fext[3 * e + 1], fz = fext[3 * e + 2];
      if (fx != 0 || fy != 0 || fz != 0) {
        m |= M_EXT;
        fextd[li] = typename VT<R>::R4{(R)fx, (R)fy, (R)fz, R(0)};
      }
    }
    meta[li] = m;
  }
}

}  // namespace vx
