// voxsim.cu -- host side of the B200 voxel stepper: lattice builder (L1),
// material tables (Eq. 1-12), step orchestration with CUDA graphs, the x-slab
// decomposition with NCCL (one slab per process) or in-process emulated
// slabs (L3), and the C ABI of include/voxsim.h (L4).
// Paper: Hiller & Lipson, arXiv:1212.2845.  Readings: DESIGN.md §3.
#include "voxsim.h"
#include "vx_kernels.cuh"
#include "vx_topology.cuh"
#include "vx_fused_yz.cuh"

#include <cub/device/device_scan.cuh>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

using namespace vx;

namespace {

// NVTX range over a scope (visible in Nsight Systems / ncu --nvtx): one per C ABI
// call that does work, per replayed graph chunk of steps, and per one-time
// phase (engine resolution, launch-geometry tuning, topology build).
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

thread_local std::string g_err;

vx_status fail(vx_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define VX_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? VX_ERR_OOM : VX_ERR_CUDA,      \
                  std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)

#define VX_NCCL(call)                                                              \
  do {                                                                             \
    ncclResult_t r_ = (call);                                                      \
    if (r_ != ncclSuccess)                                                         \
      return fail(VX_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

#define VX_TRY(call)            \
  do {                          \
    vx_status s_ = (call);      \
    if (s_ != VX_OK) return s_; \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  vx_status alloc(size_t b) {
    if (b == bytes && p) return VX_OK;
    release();
    if (b == 0) return VX_OK;
    VX_CUDA(cudaMalloc(&p, b));
    bytes = b;
    return VX_OK;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

const double kPi = 3.14159265358979323846;

inline size_t rsize(int prec) { return prec == 32 ? 4 : 8; }
inline unsigned grid_of(long long n, int b = 256) { return (unsigned)((n + b - 1) / b); }

// Balanced slab of rank r of P over nx planes: [x0, x1).
inline void slab_planes(int nx, int P, int r, int* x0, int* x1) {
  *x0 = (int)((long long)r * nx / P);
  *x1 = (int)((long long)(r + 1) * nx / P);
}

// One x-slab of the lattice: owned planes [x0, x1) plus one ghost plane on
// each side that exists, [xl0, xl1); its own SoA state and bond records.
struct Slab {
  int x0 = 0, x1 = 0, xl0 = 0, xl1 = 0;
  uint32_t nloc = 0;
  long long box_base = 0;              // xl0 * plane
  DevBuf buf[2][4];                    // state, double-buffered: [parity][pos, quat, mom, ang]
  int par = 0;                         // which copy holds the current state S_n
  DevBuf recA, recB, recC, fextd, cf, meta_d, ext_of_local;
  DevBuf sidx;                            // global surface index per local voxel (collision)
  DevBuf meta_static_d;                  // static meta bits, local box order (K1)
  // owned-voxel I/O (vx_read_state_owned): local id, global box id and position
  // in the owned order of this slab's owned voxels
  DevBuf own_lid, own_gid, own_dst;
  long long own_n = 0;
  DevBuf& pos() { return buf[par][0]; }
  DevBuf& quat() { return buf[par][1]; }
  DevBuf& mom() { return buf[par][2]; }
  DevBuf& ang() { return buf[par][3]; }
  const DevBuf& pos() const { return buf[par][0]; }
  const DevBuf& quat() const { return buf[par][1]; }
  const DevBuf& mom() const { return buf[par][2]; }
  const DevBuf& ang() const { return buf[par][3]; }
  const DevBuf& out(int a) const { return buf[par ^ 1][a]; }   // S_{n+1} of the fused step
};

}  // namespace

struct vx_lattice {
  // geometry (global)
  int nx = 0, ny = 0, nz = 0;
  double l = 0, origin[3] = {0, 0, 0};
  int prec = 32;
  int device = 0, rank = 0, nranks = 1;
  bool emulated = false;                  // nranks slabs in this process, no NCCL
  std::vector<uint8_t> cells;             // x-fastest
  uint32_t plane = 0;                     // ny * nz
  long long nbox = 0;                     // nx * plane (global)
  std::vector<Slab> slabs;                // 1 (single / NCCL rank) or nranks (emulated)
  int x0 = 0, x1 = 0;                     // planes this handle owns
  // counts (global)
  long long N = 0, nbonds = 0, nsurf = 0;
  std::vector<long long> box_of_ext;      // global box id of each external voxel
  int max_cell = 0;
  std::vector<uint8_t> pair_present;      // [256 * mat_a + mat_b] of every bond (a on the - side)
  double alpha_lo = 0, alpha_hi = 0;      // extremes of (alpha_a + alpha_b)/2 over present pairs
  // boundary (external order)
  std::vector<uint8_t> fixed;
  std::vector<double> fext;
  bool any_ext = false;
  // materials / env
  std::vector<vx_material> mats;
  bool mats_set = false, env_set = false;
  vx_env env{};
  double w2max = 0, dt = 0;
  bool tables_dirty = true;
  // device
  cudaStream_t stream = nullptr, comm_stream = nullptr;
  cudaEvent_t ev_k4 = nullptr, ev_halo = nullptr;
  DevBuf mat, pair, clk, box_of_ext_d, pair_w2, mat_w2;
  // self collision: global surface table (kernels K5 / k_contact)
  std::vector<unsigned> surf_g;           // global box id of every surface voxel, ascending
  std::vector<int> seg;                   // nranks + 1: surface segment of each rank's slab
  DevBuf surf_d, sijk, ss, cellh, bcount, bstart, bitems, rowptr, col;
  int H = 0;
  int bp_grid = 1;                        // CTAs of the cooperative broadphase
  bool ss_dirty = true;                   // the surface table must be re-packed from the state
  long long cap = 0;
  double cutoff = 0;
  // staging of the external fp64 state (vx_set_state / vx_read_state), kept between calls
  DevBuf stage_ext, stage_box;
  // owned-voxel I/O: external ids of the voxels in the owned planes, ascending,
  // and their global box ids on the device (built on first use)
  std::vector<int64_t> owned_ext;
  DevBuf owned_box_d;
  bool owned_ready = false;
  // graphs
  std::map<long long, cudaGraphExec_t> graphs;
  // instrumentation
  bool instr = false;
  int instr_stride = 1;                   // events on every instr_stride-th step
  std::vector<cudaEvent_t> events;
  double t_ms[4] = {0, 0, 0, 0};
  long long t_cnt[4] = {0, 0, 0, 0};
  // nccl
  ncclComm_t comm = nullptr;
  long long steps_done = 0;

  int engine = VX_ENGINE_FUSED;           // engine in use (provisional while AUTO is unresolved)
  int engine_req = VX_ENGINE_AUTO;        // requested (vx_set_engine); AUTO resolves at the first step
  bool engine_resolved = false;
  bool fused_smem_set[2] = {false, false};
  bool fused_yz_smem_set[2] = {false, false};
  bool yz_ok = true;                      // (y, z)-mapped fused pass for nz < 64 (VX_FUSED_YZ)
  int fused_ty = 8;                       // rows per fused block (VX_FUSED_TY overrides)
  int fused_waves = 4;                    // block waves per fused launch (VX_FUSED_WAVES)
  int fused_tune = 1;                     // time candidate segment lengths once (VX_FUSED_TUNE)
  int fused_sx = 0;                       // fixed planes per segment (VX_FUSED_SX), 0: derived
  std::map<long long, std::pair<int, int>> geo_tuned;   // (TY, SX) chosen per launch range
  int batch_stride = 0;                   // planes per batched scene (vx_set_batch)
  int batch_stride_z = 0;                 // layers per z-stacked scene (vx_set_batch_z)
  int batch_stride_y = 0;                 // rows per y-stacked scene (vx_set_batch_y)

  bool fused() const { return engine == VX_ENGINE_FUSED; }
  void flip() {
    for (auto& s : slabs) s.par ^= 1;
  }
  bool force_nccl = false;                // VX_FORCE_NCCL: the NCCL code path with one rank (tests)
  bool nccl() const { return (nranks > 1 && !emulated) || force_nccl; }
  bool collide() const { return env_set && env.self_collision && nsurf > 0; }
  // surface rows this handle builds: its rank's segment over NCCL, else all
  int rows_begin() const { return nccl() ? seg[rank] : 0; }
  int rows_end() const { return nccl() ? seg[rank + 1] : seg[nranks]; }
  // surface segment of slab q of this handle
  int slab_seg(size_t q, int end) const {
    const int r = emulated ? (int)q : rank;
    return seg[r + end];
  }
  int bond_launches() const {
    if (emulated) return (int)slabs.size();
    return nranks > 1 ? 3 : 1;
  }
  // fused launches per step: one per slab, or interior + 2 boundary planes when
  // slabs exchange ghost planes (NCCL ranks, emulated slabs)
  int fused_launches() const {
    if (!(emulated || nccl())) return (int)slabs.size();
    int k = 0;
    for (const auto& s : slabs) k += (s.x1 - s.x0) >= 3 ? 2 : 1;   // interior + boundary planes
    return k;
  }
  // clock + (surface pack and contact per slab + broadphase when colliding)
  int other_launches() const { return 1 + (collide() ? 1 + (int)slabs.size() : 0); }
  int launches_per_step() const {
    int k = 1;                                         // clock
    k += fused() ? fused_launches() : bond_launches() + (int)slabs.size();
    if (collide()) k += other_launches() - 1;
    return k;
  }
  void clear_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    graphs.clear();
  }
};

namespace {

// ---------------------------------------------------------------- L1/K1 builder
unsigned topo_grid(unsigned long long n) {
  return (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>((n + 255) / 256, 148ull * 32));
}

// out[i] = sum of in[0..i) (cub::DeviceScan, setup only)
vx_status exclusive_scan_u32(const uint32_t* in, uint32_t* out, unsigned long long n, cudaStream_t st) {
  size_t tmp = 0;
  VX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int64_t)n, st));
  DevBuf t;
  VX_TRY(t.alloc(std::max<size_t>(tmp, 16)));
  VX_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, (int64_t)n, st));
  return VX_OK;
}

// External ids, static meta of every slab, counts, material-pair table and
// the surface list, built on the device from the grid (vx_topology.cuh).
vx_status build_topology(vx_lattice* h) {
  Nvtx nvtx_("vx build topology (K1)");
  const int nx = h->nx, ny = h->ny, nz = h->nz;
  const unsigned long long nbox = (unsigned long long)h->nbox;
  cudaStream_t st = h->stream;
  DevBuf cells_d, flag, scan, counts, pairs, maxc;
  VX_TRY(cells_d.alloc(nbox));
  VX_CUDA(cudaMemcpyAsync(cells_d.p, h->cells.data(), nbox, cudaMemcpyHostToDevice, st));
  VX_TRY(flag.alloc(nbox * 4));
  VX_TRY(scan.alloc(nbox * 4));
  const uint8_t* cd = cells_d.as<uint8_t>();
  // external ids: filled cells in x-fastest order (vx_lattice_desc.cells)
  k_topo_filled<<<topo_grid(nbox), 256, 0, st>>>(cd, nbox, flag.as<uint32_t>());
  VX_TRY(exclusive_scan_u32(flag.as<uint32_t>(), scan.as<uint32_t>(), nbox, st));
  uint32_t last[2] = {0, 0};
  VX_CUDA(cudaMemcpyAsync(&last[0], scan.as<uint32_t>() + (nbox - 1), 4, cudaMemcpyDeviceToHost, st));
  VX_CUDA(cudaMemcpyAsync(&last[1], flag.as<uint32_t>() + (nbox - 1), 4, cudaMemcpyDeviceToHost, st));
  VX_CUDA(cudaStreamSynchronize(st));
  h->N = (long long)last[0] + last[1];
  VX_TRY(h->box_of_ext_d.alloc((size_t)std::max<long long>(h->N, 1) * 8));
  k_topo_ext<<<topo_grid(nbox), 256, 0, st>>>(cd, nx, ny, nz, nbox, scan.as<uint32_t>(),
                                              h->box_of_ext_d.as<long long>());
  h->box_of_ext.resize((size_t)h->N);
  if (h->N)
    VX_CUDA(cudaMemcpyAsync(h->box_of_ext.data(), h->box_of_ext_d.p, (size_t)h->N * 8, cudaMemcpyDeviceToHost, st));
  // counts, pair table, surface flags (reusing `flag`)
  VX_TRY(counts.alloc(16));
  VX_TRY(pairs.alloc(2048 * 4));
  VX_TRY(maxc.alloc(4));
  VX_CUDA(cudaMemsetAsync(counts.p, 0, 16, st));
  VX_CUDA(cudaMemsetAsync(pairs.p, 0, 2048 * 4, st));
  VX_CUDA(cudaMemsetAsync(maxc.p, 0, 4, st));
  k_topo_count<<<std::min(topo_grid(nbox), 148u * 4), 256, 0, st>>>(cd, nx, ny, nz, nbox, counts.as<unsigned long long>(),
                                                pairs.as<unsigned>(), maxc.as<int>(), flag.as<uint32_t>());
  VX_TRY(exclusive_scan_u32(flag.as<uint32_t>(), scan.as<uint32_t>(), nbox, st));
  unsigned long long cnt[2];
  std::vector<unsigned> pb(2048);
  VX_CUDA(cudaMemcpyAsync(cnt, counts.p, 16, cudaMemcpyDeviceToHost, st));
  VX_CUDA(cudaMemcpyAsync(pb.data(), pairs.p, 2048 * 4, cudaMemcpyDeviceToHost, st));
  VX_CUDA(cudaMemcpyAsync(&h->max_cell, maxc.p, 4, cudaMemcpyDeviceToHost, st));
  VX_CUDA(cudaStreamSynchronize(st));
  h->nbonds = (long long)cnt[0];
  h->nsurf = (long long)cnt[1];
  h->pair_present.assign(256 * 256, 0);
  for (int x = 0; x < 65536; ++x)
    if (pb[x >> 5] & (1u << (x & 31))) h->pair_present[x] = 1;
  // surface list (global box ids, ascending)
  h->surf_g.resize((size_t)h->nsurf);
  if (h->nsurf) {
    DevBuf sg;
    VX_TRY(sg.alloc((size_t)h->nsurf * 4));
    k_topo_surf<<<topo_grid(nbox), 256, 0, st>>>(flag.as<uint32_t>(), scan.as<uint32_t>(), nbox, sg.as<unsigned>());
    VX_CUDA(cudaMemcpyAsync(h->surf_g.data(), sg.p, (size_t)h->nsurf * 4, cudaMemcpyDeviceToHost, st));
    VX_CUDA(cudaStreamSynchronize(st));
  }
  // static meta of every slab's local box: material, filled, neighbour mask, surface
  for (auto& s : h->slabs) {
    VX_TRY(s.meta_static_d.alloc((size_t)s.nloc * 4));
    k_topo_meta<<<grid_of(s.nloc), 256, 0, st>>>(cd, nx, ny, nz, s.xl0, s.nloc, s.meta_static_d.as<uint32_t>());
  }
  VX_CUDA(cudaGetLastError());
  VX_CUDA(cudaStreamSynchronize(st));
  // surface segment of every rank's slab (box order is x-slowest)
  h->seg.assign((size_t)h->nranks + 1, 0);
  for (int r = 0; r < h->nranks; ++r) {
    int a, b;
    slab_planes(nx, h->nranks, r, &a, &b);
    h->seg[r] = (int)(std::lower_bound(h->surf_g.begin(), h->surf_g.end(), (unsigned)a * h->plane) - h->surf_g.begin());
    h->seg[r + 1] = (int)(std::lower_bound(h->surf_g.begin(), h->surf_g.end(), (unsigned)b * h->plane) - h->surf_g.begin());
  }
  return VX_OK;
}

template <class R> Dev<R> make_dev(const vx_lattice* h, const Slab& s) {
  Dev<R> d;
  d.pos = s.pos().as<typename VT<R>::R4>();
  d.quat = s.quat().as<typename VT<R>::R4>();
  d.mom = s.mom().as<typename VT<R>::R4>();
  d.ang = s.ang().as<typename VT<R>::R2>();
  d.recA = s.recA.as<typename VT<R>::R4>();
  d.recB = s.recB.as<typename VT<R>::R4>();
  d.recC = s.recC.as<R>();
  d.fext = h->any_ext ? s.fextd.as<typename VT<R>::R4>() : nullptr;
  d.cf = s.cf.as<typename VT<R>::R4>();
  d.sidx = s.sidx.as<int>();
  d.ss = h->ss.as<typename VT<R>::R4>();
  d.mat = h->mat.as<MatC<R>>();
  d.pair = h->pair.as<PairC<R>>();
  d.clk = h->clk.as<Clock>();
  d.nmat = (int)h->mats.size();
  d.nloc = s.nloc;
  d.sx = h->plane;
  d.ny = (uint32_t)h->ny;
  d.nz = (uint32_t)h->nz;
  d.xl0 = s.xl0;
  d.l = (R)h->l;
  d.half_l = (R)(0.5 * h->l);
  d.dt = (R)h->dt;
  d.l_d = h->l;
  d.zbase_d = h->origin[2] - h->env.floor_z;
  d.bz = (uint32_t)h->batch_stride_z;
  d.floor_on = h->env_set ? h->env.floor_on : 0;
  d.ground = (h->env_set && h->env.zeta_ground > 0) ? 1 : 0;
  return d;
}

vx_status upload_meta(vx_lattice* h) {
  // static bits + boundary bits (FIXED, EXT) -> device, merged with the latch bits
  const bool any_fixed = std::any_of(h->fixed.begin(), h->fixed.end(), [](uint8_t v) { return v != 0; });
  DevBuf fx, fe;
  if (any_fixed) {
    VX_TRY(fx.alloc((size_t)h->N));
    VX_CUDA(cudaMemcpyAsync(fx.p, h->fixed.data(), (size_t)h->N, cudaMemcpyHostToDevice, h->stream));
  }
  if (h->any_ext) {
    VX_TRY(fe.alloc((size_t)h->N * 24));
    VX_CUDA(cudaMemcpyAsync(fe.p, h->fext.data(), (size_t)h->N * 24, cudaMemcpyHostToDevice, h->stream));
  }
  for (auto& s : h->slabs) {
    VX_CUDA(cudaMemcpyAsync(s.meta_d.p, s.meta_static_d.p, (size_t)s.nloc * 4, cudaMemcpyDeviceToDevice, h->stream));
    if (h->any_ext) {
      VX_TRY(s.fextd.alloc((size_t)s.nloc * 4 * rsize(h->prec)));
      VX_CUDA(cudaMemsetAsync(s.fextd.p, 0, s.fextd.bytes, h->stream));
    }
    if ((any_fixed || h->any_ext) && h->N) {
      const unsigned g = topo_grid((unsigned long long)h->N);
      if (h->prec == 32)
        k_apply_bc<float><<<g, 256, 0, h->stream>>>(h->box_of_ext_d.as<long long>(), h->N, s.box_base, s.nloc,
                                                    fx.as<uint8_t>(), fe.as<double>(), s.meta_d.as<uint32_t>(),
                                                    s.fextd.as<float4>());
      else
        k_apply_bc<double><<<g, 256, 0, h->stream>>>(h->box_of_ext_d.as<long long>(), h->N, s.box_base, s.nloc,
                                                     fx.as<uint8_t>(), fe.as<double>(), s.meta_d.as<uint32_t>(),
                                                     s.fextd.as<double4>());
    }
    if (h->prec == 32)
      k_merge_meta<float><<<grid_of(s.nloc), 256, 0, h->stream>>>(make_dev<float>(h, s), s.meta_d.as<uint32_t>(), s.nloc);
    else
      k_merge_meta<double><<<grid_of(s.nloc), 256, 0, h->stream>>>(make_dev<double>(h, s), s.meta_d.as<uint32_t>(), s.nloc);
    VX_CUDA(cudaGetLastError());
  }
  VX_CUDA(cudaStreamSynchronize(h->stream));
  h->clear_graphs();
  return VX_OK;
}

// ---------------------------------------------------------------- tables
struct MatD {
  double E, nu, rho, cte, mu_s, mu_d, G, m, I;
};
MatD mat_d(const vx_material& v, double l) {
  MatD m{v.E, v.nu, v.rho, v.cte, v.mu_s, v.mu_d, 0, 0, 0};
  m.G = v.E / (2 * (1 + v.nu));
  m.m = v.rho * l * l * l;        // voxel mass
  m.I = m.m * l * l / 6.0;        // R8: solid cube
  return m;
}
// Eq. 1-12 for the pair (a, b)
void pair_consts(const MatD& a, const MatD& b, double l, double* a1, double* a2, double* b1,
                 double* b2, double* b3) {
  const double Ec = 2 * a.E * b.E / (a.E + b.E);   // Eq. 1
  const double Gc = 2 * a.G * b.G / (a.G + b.G);   // Eq. 2
  const double A = l * l, I = l * l * l * l / 12.0, J = l * l * l * l / 6.0;  // Eq. 4-5
  *a1 = Ec * A / l;                                 // Eq. 8
  *a2 = Gc * J / l;                                 // Eq. 9
  *b1 = 12 * Ec * I / (l * l * l);                  // Eq. 10
  *b2 = 6 * Ec * I / (l * l);                       // Eq. 11
  *b3 = 2 * Ec * I / l;                             // Eq. 12
}

template <class R> vx_status upload_tables(vx_lattice* h) {
  const int n = (int)h->mats.size();
  const double l = h->l, dt = h->dt;
  const vx_env& e = h->env;
  std::vector<MatC<R>> mc(n);
  std::vector<PairC<R>> pc((size_t)n * n);
  std::vector<MatD> md(n);
  for (int i = 0; i < n; ++i) md[i] = mat_d(h->mats[i], l);
  h->alpha_lo = 0;
  h->alpha_hi = 0;
  for (int i = 0; i < n; ++i) {
    const MatD& m = md[i];
    MatC<R>& c = mc[i];
    c.m = (R)m.m;
    c.inv_m = (R)(1.0 / m.m);
    c.inv_I = (R)(1.0 / m.I);
    c.dt_m = (R)(dt / m.m);
    c.dt_I = (R)(dt / m.I);
    c.mg = (R)(m.m * e.gravity);
    c.cgt = (R)(2 * e.zeta_ground * std::sqrt(m.m * m.E * l));
    c.cgr = (R)(2 * e.zeta_ground * std::sqrt(m.I * m.G * l * l * l / 6.0));
    c.kf = (R)(m.E * l);
    c.cfl = (R)(2 * e.zeta_col * std::sqrt(m.m * m.E * l));
    c.alpha = (R)m.cte;
    c.mu_s = (R)m.mu_s;
    c.mu_d = (R)m.mu_d;
    c.kc = (R)(m.E * l);
    c.pad0 = c.pad1 = (R)0;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double a1, a2, b1, b2, b3;
      pair_consts(md[i], md[j], l, &a1, &a2, &b1, &b2, &b3);
      PairC<R>& p = pc[(size_t)i * n + j];
      p.a1 = (R)a1; p.a2 = (R)a2; p.b1 = (R)b1; p.b2 = (R)b2; p.nb2 = -(R)b2; p.b3 = (R)b3;
      p.alpha_mean = (R)(0.5 * (md[i].cte + md[j].cte));
      const double mmin = std::min(md[i].m, md[j].m), Imin = std::min(md[i].I, md[j].I);
      const double ct = 2 * e.zeta_bond * std::sqrt(mmin * a1);   // Eq. 34, R10
      const double cr = 2 * e.zeta_bond * std::sqrt(Imin * a2);   // Eq. 35, R11
      p.ct2 = (R)(0.5 * ct);
      p.ct4 = (R)(0.25 * ct);
      p.cr2 = (R)(0.5 * cr);
      p.inv_m_b = (R)(1.0 / md[j].m);
      p.inv_I_b = (R)(1.0 / md[j].I);
      if (h->pair_present[(size_t)i * 256 + j]) {   // Eq. 40 fault bounds
        h->alpha_lo = std::min(h->alpha_lo, 0.5 * (md[i].cte + md[j].cte));
        h->alpha_hi = std::max(h->alpha_hi, 0.5 * (md[i].cte + md[j].cte));
      }
    }
  VX_TRY(h->mat.alloc(mc.size() * sizeof(MatC<R>)));
  VX_TRY(h->pair.alloc(pc.size() * sizeof(PairC<R>)));
  VX_CUDA(cudaMemcpy(h->mat.p, mc.data(), mc.size() * sizeof(MatC<R>), cudaMemcpyHostToDevice));
  VX_CUDA(cudaMemcpy(h->pair.p, pc.data(), pc.size() * sizeof(PairC<R>), cudaMemcpyHostToDevice));
  return VX_OK;
}

// K2: stable timestep from a device max-reduction (Eq. 31-32, R9)
template <class R> vx_status compute_dt(vx_lattice* h) {
  const int n = (int)h->mats.size();
  std::vector<MatD> md(n);
  for (int i = 0; i < n; ++i) md[i] = mat_d(h->mats[i], h->l);
  std::vector<double> pw((size_t)n * n), mw(n);
  for (int i = 0; i < n; ++i) {
    mw[i] = md[i].E * h->l / md[i].m;
    for (int j = 0; j < n; ++j) {
      double a1, a2, b1, b2, b3;
      pair_consts(md[i], md[j], h->l, &a1, &a2, &b1, &b2, &b3);
      pw[(size_t)i * n + j] = a1 / std::min(md[i].m, md[j].m);
    }
  }
  VX_TRY(h->pair_w2.alloc(pw.size() * 8));
  VX_TRY(h->mat_w2.alloc(mw.size() * 8));
  VX_CUDA(cudaMemcpy(h->pair_w2.p, pw.data(), pw.size() * 8, cudaMemcpyHostToDevice));
  VX_CUDA(cudaMemcpy(h->mat_w2.p, mw.data(), mw.size() * 8, cudaMemcpyHostToDevice));
  Clock* c = h->clk.as<Clock>();
  VX_CUDA(cudaMemsetAsync(&c->w2_bond_bits, 0, 16, h->stream));
  for (auto& s : h->slabs) {
    // planes [xl0, x1): the right ghost plane's +x bonds belong to the next slab
    // (its +x neighbour is outside this slab's box)
    const uint32_t end = (uint32_t)(s.x1 - s.xl0) * h->plane;
    k_dt<R><<<grid_of(end), 256, 0, h->stream>>>(s.pos().as<typename VT<R>::R4>(), 0u, end,
                                                 h->plane, (uint32_t)h->nz, h->pair_w2.as<double>(),
                                                 h->mat_w2.as<double>(), n, c);
  }
  VX_CUDA(cudaGetLastError());
  unsigned long long bits[2];
  VX_CUDA(cudaMemcpyAsync(bits, &c->w2_bond_bits, 16, cudaMemcpyDeviceToHost, h->stream));
  VX_CUDA(cudaStreamSynchronize(h->stream));
  double wb, wv;
  std::memcpy(&wb, &bits[0], 8);
  std::memcpy(&wv, &bits[1], 8);
  if (h->nccl()) {
    DevBuf t;
    VX_TRY(t.alloc(16));
    double hv[2] = {wb, wv};
    VX_CUDA(cudaMemcpy(t.p, hv, 16, cudaMemcpyHostToDevice));
    VX_NCCL(ncclAllReduce(t.p, t.p, 2, ncclDouble, ncclMax, h->comm, h->stream));
    VX_CUDA(cudaMemcpyAsync(hv, t.p, 16, cudaMemcpyDeviceToHost, h->stream));
    VX_CUDA(cudaStreamSynchronize(h->stream));
    wb = hv[0];
    wv = hv[1];
  }
  // omega_0m: max over bonds; a lattice without bonds falls back to E l / m
  h->w2max = h->nbonds > 0 ? wb : wv;
  return VX_OK;
}

void update_dt(vx_lattice* h) {
  const double s = h->env_set ? h->env.dt_safety : 1.0;
  h->dt = h->w2max > 0 ? s / (2 * kPi * std::sqrt(h->w2max)) : 0.0;
}

vx_status setup_collision(vx_lattice* h) {
  const int S = (int)h->surf_g.size();
  const size_t r = rsize(h->prec);
  VX_TRY(h->surf_d.alloc((size_t)std::max(S, 1) * 4));
  if (S) VX_CUDA(cudaMemcpy(h->surf_d.p, h->surf_g.data(), (size_t)S * 4, cudaMemcpyHostToDevice));
  {   // lattice coordinates of every surface entry (the contact kernel's table)
    std::vector<int4> ijk((size_t)std::max(S, 1));
    for (int s = 0; s < S; ++s) {
      const unsigned g = h->surf_g[s];
      ijk[s] = make_int4((int)(g / h->plane), (int)((g / h->nz) % h->ny), (int)(g % h->nz), 0);
    }
    VX_TRY(h->sijk.alloc(ijk.size() * sizeof(int4)));
    VX_CUDA(cudaMemcpy(h->sijk.p, ijk.data(), ijk.size() * sizeof(int4), cudaMemcpyHostToDevice));
  }
  VX_TRY(h->ss.alloc((size_t)std::max(S, 1) * 2 * 4 * r));
  int H = 1024;
  while (H < 2 * S) H <<= 1;
  h->H = H;
  {   // cooperative broadphase grid: resident CTAs, no more than the work needs
    int per_sm = 0, sms = 0;
    VX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, h->prec == 32 ? (const void*)k_broadphase<float> : (const void*)k_broadphase<double>, 1024, 0));
    VX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    h->bp_grid = std::max(1, std::min(std::max(1, per_sm) * sms, (std::max(S * BP_LANES, H) + 1023) / 1024));
  }
  const int rows = h->rows_end() - h->rows_begin();
  h->cap = std::max<long long>(1 << 16, 128LL * rows);
  VX_TRY(h->cellh.alloc((size_t)std::max(S, 1) * sizeof(int4)));
  VX_TRY(h->bcount.alloc((size_t)H * 4));
  VX_TRY(h->bstart.alloc((size_t)(H + 1) * 4));
  VX_TRY(h->bitems.alloc((size_t)std::max(S, 1) * 4));
  VX_TRY(h->rowptr.alloc((size_t)(S + 1) * 4));
  VX_TRY(h->col.alloc((size_t)h->cap * 4));
  VX_CUDA(cudaMemset(h->rowptr.p, 0, (size_t)(S + 1) * 4));
  for (size_t q = 0; q < h->slabs.size(); ++q) {
    Slab& sl = h->slabs[q];
    VX_TRY(sl.cf.alloc((size_t)sl.nloc * 4 * r));
    VX_CUDA(cudaMemset(sl.cf.p, 0, sl.cf.bytes));
    std::vector<int> si(sl.nloc, -1);
    for (int s = h->slab_seg(q, 0); s < h->slab_seg(q, 1); ++s)
      si[(size_t)((long long)h->surf_g[s] - sl.box_base)] = s;
    VX_TRY(sl.sidx.alloc((size_t)sl.nloc * 4));
    VX_CUDA(cudaMemcpy(sl.sidx.p, si.data(), (size_t)sl.nloc * 4, cudaMemcpyHostToDevice));
  }
  h->ss_dirty = true;
  // cutoff = 2 r_max + horizon, r_max = (l/2)(1 + max|alpha| |T_amp|)
  double amax = 0;
  for (auto& m : h->mats) amax = std::max(amax, std::fabs(m.cte));
  const double rmax = 0.5 * h->l * (1 + amax * std::fabs(h->env.T_amp));
  h->cutoff = 2 * rmax + h->env.horizon_voxels * h->l;
  return VX_OK;
}

vx_status prepare(vx_lattice* h) {
  if (!h->fused()) {   // bond records (K3 -> K4), allocated on the first two-pass step
    const size_t r = rsize(h->prec);
    for (Slab& sl : h->slabs) {
      if (sl.recA.p) continue;
      const size_t n = sl.nloc;
      VX_TRY(sl.recA.alloc(3 * n * 4 * r));
      VX_TRY(sl.recB.alloc(3 * n * 4 * r));
      VX_TRY(sl.recC.alloc(3 * n * r));
      VX_CUDA(cudaMemset(sl.recA.p, 0, sl.recA.bytes));
      VX_CUDA(cudaMemset(sl.recB.p, 0, sl.recB.bytes));
      VX_CUDA(cudaMemset(sl.recC.p, 0, sl.recC.bytes));
      h->clear_graphs();
    }
  }
  if (!h->mats_set) return fail(VX_ERR_STATE, "vx_set_materials has not been called");
  if (!h->env_set) return fail(VX_ERR_STATE, "vx_set_environment has not been called");
  if (h->tables_dirty) {
    update_dt(h);
    if (h->prec == 32) VX_TRY(upload_tables<float>(h));
    else VX_TRY(upload_tables<double>(h));
    if (h->collide()) VX_TRY(setup_collision(h));
    h->tables_dirty = false;
    h->clear_graphs();
  }
  return VX_OK;
}

// ---------------------------------------------------------------- one step
template <class R>
void launch_bonds(vx_lattice* h, const Slab& s, const Dev<R>& d, int p0, int p1) {
  if (p1 <= p0) return;
  const uint32_t beg = (uint32_t)(p0 - s.xl0) * h->plane, end = (uint32_t)(p1 - s.xl0) * h->plane;
  k_bonds<R><<<grid_of(end - beg), 256, 0, h->stream>>>(d, beg, end);
}

template <class R> void launch_integrate(vx_lattice* h, const Slab& s, const Dev<R>& d, bool col) {
  const uint32_t beg = (uint32_t)(s.x0 - s.xl0) * h->plane, end = (uint32_t)(s.x1 - s.xl0) * h->plane;
  if (col)
    k_integrate<R, true><<<grid_of(end - beg), 256, 0, h->stream>>>(d, beg, end, s.ext_of_local.as<uint32_t>());
  else
    k_integrate<R, false><<<grid_of(end - beg), 256, 0, h->stream>>>(d, beg, end, s.ext_of_local.as<uint32_t>());
}

inline long long fused_key(const Slab& s, int x_begin, int x_end) {
  return ((long long)s.x0 << 40) | ((long long)x_begin << 20) | (long long)x_end;
}

template <class R>
vx_status launch_fused(vx_lattice* h, const Slab& s, bool col, int x_begin, int x_end, int sx_force = 0,
                       cudaStream_t st = nullptr, int x_begin2 = 0, int x_end2 = 0, int ty_force = 0);

// Launch-geometry tuning of the fused pass (once per launch range, outside any
// graph).  The step time depends on rows per block (TY) and planes per block
// segment (SX): the -y / -x halos cost 1/TY and 1/SX extra bonds, a block's
// rows are a serial chain (small lattices want many one-row blocks, TY = SX =
// 1: C4 22 -> 7 us/step), and the block count sets the wave quantisation over
// 148 SMs x 2 resident blocks -- in a way no closed rule captured
// (profiles/r07_tuning.md).  Each candidate recomputes S_{n+1} from S_n into
// the spare copy; the arithmetic per voxel is the same for every geometry
// (explicit rounding, tests/test_gpu_geometry.py), so the state the real step
// then writes is unchanged.  VX_FUSED_TY / VX_FUSED_WAVES fix the geometry.
template <class R> vx_status tune_fused(vx_lattice* h) {
  Nvtx nvtx_("vx tune fused geometry");
  if (!h->fused() || h->fused_tune == 0 || !h->geo_tuned.empty()) return VX_OK;
  const bool split = h->emulated || h->nccl();
  const bool col = h->collide();
  Clock saved;   // the candidates' motion-budget / divergence atomics must not leak
  VX_CUDA(cudaMemcpy(&saved, h->clk.p, sizeof saved, cudaMemcpyDeviceToHost));
  struct Ev {   // released on every exit path
    cudaEvent_t e = nullptr;
    ~Ev() { if (e) cudaEventDestroy(e); }
  } ev0, ev1;
  VX_CUDA(cudaEventCreate(&ev0.e));
  VX_CUDA(cudaEventCreate(&ev1.e));
  const cudaEvent_t e0 = ev0.e, e1 = ev1.e;
  for (const Slab& s : h->slabs) {
    const int b = split ? s.x0 + 1 : s.x0, e = split ? s.x1 - 1 : s.x1;
    const int planes = e - b;
    if (planes < 1) continue;
    const bool big = (long long)planes * h->plane >= (1LL << 22);
    static const int ty_big[] = {4, 5, 6, 7, 8}, ty_small[] = {1, 2, 4, 5, 6, 7, 8};
    static const int sx_big[] = {3, 4, 5, 6, 7, 8, 10, 12, 14, 16, 20, 24, 32};
    static const int sx_small[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32};
    const int* tys = big ? ty_big : ty_small;
    const int nty = big ? 5 : 7;
    const int* sxs = big ? sx_big : sx_small;
    const int nsx = big ? 13 : 10;
    const int reps = big ? 3 : 8;
    auto time_geo = [&](int ty, int sx, int nrep, float* ms) -> vx_status {
      VX_TRY(launch_fused<R>(h, s, col, b, e, sx, nullptr, 0, 0, ty));   // warm
      VX_CUDA(cudaEventRecord(e0, h->stream));
      for (int r = 0; r < nrep; ++r) VX_TRY(launch_fused<R>(h, s, col, b, e, sx, nullptr, 0, 0, ty));
      VX_CUDA(cudaEventRecord(e1, h->stream));
      VX_CUDA(cudaEventSynchronize(e1));
      VX_CUDA(cudaEventElapsedTime(ms, e0, e1));
      *ms /= (float)nrep;
      return VX_OK;
    };
    std::vector<std::pair<float, std::pair<int, int>>> times;
    for (int a = 0; a < nty; ++a) {
      const int ty = tys[a];
      if (ty > h->ny && ty != tys[0]) break;
      for (int c = 0; c < nsx; ++c) {
        const int sx = sxs[c];
        if (sx > planes && c > 0) break;
        float ms = 0;
        VX_TRY(time_geo(ty, sx, reps, &ms));
        times.push_back({ms, {ty, sx}});
      }
    }
    if (times.empty()) continue;
    // second round: the six fastest re-timed with three times the repetitions
    std::sort(times.begin(), times.end());
    if (times.size() > 6) times.resize(6);
    for (auto& c : times) VX_TRY(time_geo(c.second.first, c.second.second, 3 * reps, &c.first));
    // fastest; a smaller TY within 0.3 % (a tie) wins: shorter row tiles re-read
    // fewer neighbour rows from DRAM (profiles/r09_geometry.md)
    float best = 1e30f;
    for (auto& c : times) best = std::min(best, c.first);
    std::pair<int, int> best_g{0, 0};
    float best_t = 1e30f;
    for (auto& c : times) {
      if (c.first > 1.003f * best) continue;
      if (!best_g.first || c.second.first < best_g.first ||
          (c.second.first == best_g.first && c.first < best_t)) {
        best_g = c.second;
        best_t = c.first;
      }
    }
    h->geo_tuned[fused_key(s, b, e)] = best_g;
    if (std::getenv("VX_FUSED_TUNE_LOG"))
      std::fprintf(stderr, "voxsim: fused geometry for planes [%d, %d): TY=%d SX=%d (%.3f ms / launch)\n", b, e,
                   best_g.first, best_g.second, best_t);
  }
  VX_CUDA(cudaMemcpy(h->clk.p, &saved, sizeof saved, cudaMemcpyHostToDevice));
  h->ss_dirty = true;   // the candidates wrote S_{n+1} entries into the surface table
  if (h->geo_tuned.empty()) h->geo_tuned[-1] = {0, 0};   // nothing to tune: do not retry
  h->clear_graphs();
  return VX_OK;
}

// Fused single pass over a slab's owned planes: S_n (current copy) -> S_{n+1}
// (other copy).  Block = one thread per z (a chunk of <= 256) x TY rows x SX planes.
template <class R>
vx_status launch_fused(vx_lattice* h, const Slab& s, bool col, int x_begin, int x_end, int sx_force,
                       cudaStream_t st, int x_begin2, int x_end2, int ty_force) {
  if (x_end <= x_begin) return VX_OK;
  if (!st) st = h->stream;
  const Dev<R> d = make_dev<R>(h, s);
  FusedArgs<R> a;
  a.opos = s.out(0).as<typename VT<R>::R4>();
  a.oquat = s.out(1).as<typename VT<R>::R4>();
  a.omom = s.out(2).as<typename VT<R>::R4>();
  a.oang = s.out(3).as<typename VT<R>::R2>();
  a.ext_of_local = s.ext_of_local.as<uint32_t>();
  a.p0 = x_begin - s.xl0;
  a.p1 = x_end - s.xl0;
  a.nplanes = s.xl1 - s.xl0;
  // one thread per z, in chunks of at most 256 (taller lattices: several z
  // chunks, each recomputing its lowest -z bond)
  const int threads = std::min(256, ((h->nz + 31) / 32) * 32);
  a.zchunks = (h->nz + threads - 1) / threads;
  // rows per block and planes per segment: forced (tuning, boundary planes),
  // tuned for this range, or the defaults
  const auto tuned = h->geo_tuned.find(fused_key(s, x_begin, x_end));
  const bool have = tuned != h->geo_tuned.end() && tuned->second.first > 0;
  if (h->yz_ok && h->nz < 64 && h->ny >= 2) {
    // shallow lattice: G rows side by side (vx_fused_yz.cuh); "TY" counts steps of G rows
    const int G = std::min(h->ny, 256 / h->nz);
    const int nthr = ((G * h->nz + 31) / 32) * 32;
    const int mult = ty_force > 0 ? ty_force : (have ? tuned->second.first : h->fused_ty);
    a.ty = std::min(h->ny, G * std::max(1, mult));
    a.zchunks = G;
    a.ntiles_y = (h->ny + a.ty - 1) / a.ty;
    const int planes = a.p1 - a.p0;
    const int target = 148 * 2 * h->fused_waves;
    const int nseg = std::max(1, std::min(planes, (target + a.ntiles_y - 1) / a.ntiles_y));
    a.sx = (planes + nseg - 1) / nseg;
    if (sx_force > 0) a.sx = std::min(sx_force, planes);
    else if (have) a.sx = std::min(tuned->second.second, planes);
    else if (h->fused_sx > 0) a.sx = std::min(h->fused_sx, planes);
    const int segs = (planes + a.sx - 1) / a.sx;
    const int pi = sizeof(R) == 4 ? 0 : 1;
    if (!h->fused_yz_smem_set[pi]) {
      VX_CUDA(cudaFuncSetAttribute(k_step_fused_yz<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      VX_CUDA(cudaFuncSetAttribute(k_step_fused_yz<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      h->fused_yz_smem_set[pi] = true;
    }
    a.nblk0 = a.ntiles_y * segs;
    a.p0b = a.p1b = 0;
    int segs2 = 0;
    if (x_end2 > x_begin2) {
      a.p0b = x_begin2 - s.xl0;
      a.p1b = x_end2 - s.xl0;
      segs2 = (a.p1b - a.p0b + a.sx - 1) / a.sx;
    }
    const unsigned grid = (unsigned)(a.ntiles_y * (segs + segs2));
    const size_t smem = fused_yz_smem<R>(a.ty, h->nz, G);
    if (col) k_step_fused_yz<R, true><<<grid, nthr, smem, st>>>(d, a);
    else k_step_fused_yz<R, false><<<grid, nthr, smem, st>>>(d, a);
    return VX_OK;
  }
  int ty = std::min(ty_force > 0 ? ty_force : (have ? tuned->second.first : h->fused_ty), h->ny);
  a.ty = ty;
  a.ntiles_y = (h->ny + a.ty - 1) / a.ty;
  const int planes = a.p1 - a.p0;
  const int target = 148 * 2 * h->fused_waves;   // blocks: waves at 2 resident blocks per SM
  const int nseg = std::max(1, std::min(planes, (target + a.ntiles_y - 1) / a.ntiles_y));
  a.sx = (planes + nseg - 1) / nseg;
  if (sx_force > 0) a.sx = std::min(sx_force, planes);
  else if (have) a.sx = std::min(tuned->second.second, planes);
  else if (h->fused_sx > 0) a.sx = std::min(h->fused_sx, planes);
  const int segs = (planes + a.sx - 1) / a.sx;
  const int pi = sizeof(R) == 4 ? 0 : 1;
  if (!h->fused_smem_set[pi]) {
    VX_CUDA(cudaFuncSetAttribute(k_step_fused<R, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    VX_CUDA(cudaFuncSetAttribute(k_step_fused<R, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    VX_CUDA(cudaFuncSetAttribute(k_step_fused<R, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    VX_CUDA(cudaFuncSetAttribute(k_step_fused<R, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    h->fused_smem_set[pi] = true;
  }
  a.nblk0 = a.ntiles_y * segs * a.zchunks;
  a.p0b = a.p1b = 0;
  int segs2 = 0;
  if (x_end2 > x_begin2) {   // second range, same segment length and rows per block
    a.p0b = x_begin2 - s.xl0;
    a.p1b = x_end2 - s.xl0;
    segs2 = (a.p1b - a.p0b + a.sx - 1) / a.sx;
  }
  const unsigned grid = (unsigned)(a.ntiles_y * (segs + segs2) * a.zchunks);
  const size_t smem = fused_smem<R>(a.ty, threads);
  if (a.zchunks > 1) {
    if (col) k_step_fused<R, true, true><<<grid, threads, smem, st>>>(d, a);
    else k_step_fused<R, false, true><<<grid, threads, smem, st>>>(d, a);
  } else {
    if (col) k_step_fused<R, true, false><<<grid, threads, smem, st>>>(d, a);
    else k_step_fused<R, false, false><<<grid, threads, smem, st>>>(d, a);
  }
  return VX_OK;
}

// A slab's first and last owned planes (they read the ghost planes) in one
// launch: one plane per segment, TY chosen for about one wave of blocks.
template <class R> vx_status launch_boundary(vx_lattice* h, const Slab& s, bool col, cudaStream_t st) {
  const int w = s.x1 - s.x0;
  const int nb = w >= 2 ? 2 : 1;
  const int ty = std::max(1, std::min(h->fused_ty, (h->ny * nb + 295) / 296));
  if (w <= 2) return launch_fused<R>(h, s, col, s.x0, s.x1, 1, st, 0, 0, ty);
  return launch_fused<R>(h, s, col, s.x0, s.x0 + 1, 1, st, s.x1 - 1, s.x1, ty);
}

// The four SoA state arrays of a slab, with element sizes.
struct Arr {
  char* base;
  size_t esz;
};
void state_arrays(const vx_lattice* h, const Slab& s, Arr out[4]) {
  const size_t r = rsize(h->prec);
  out[0] = {s.pos().as<char>(), 4 * r};
  out[1] = {s.quat().as<char>(), 4 * r};
  out[2] = {s.mom().as<char>(), 4 * r};
  out[3] = {s.ang().as<char>(), 2 * r};
}
inline char* plane_ptr(const Arr& a, const Slab& s, int x, size_t plane) {
  return a.base + (size_t)(x - s.xl0) * plane * a.esz;
}

// NCCL ghost exchange of state S_n (one slab per rank), on comm_stream
vx_status halo_nccl(vx_lattice* h) {
  const Slab& s = h->slabs[0];
  Arr arrs[4];
  state_arrays(h, s, arrs);
  VX_NCCL(ncclGroupStart());
  for (auto& a : arrs) {
    const size_t bytes = h->plane * a.esz;
    if (s.x0 > 0) {   // left neighbour: send my first owned plane, receive my left ghost
      VX_NCCL(ncclSend(plane_ptr(a, s, s.x0, h->plane), bytes, ncclInt8, h->rank - 1, h->comm, h->comm_stream));
      VX_NCCL(ncclRecv(plane_ptr(a, s, s.x0 - 1, h->plane), bytes, ncclInt8, h->rank - 1, h->comm, h->comm_stream));
    }
    if (s.x1 < h->nx) {   // right neighbour
      VX_NCCL(ncclSend(plane_ptr(a, s, s.x1 - 1, h->plane), bytes, ncclInt8, h->rank + 1, h->comm, h->comm_stream));
      VX_NCCL(ncclRecv(plane_ptr(a, s, s.x1, h->plane), bytes, ncclInt8, h->rank + 1, h->comm, h->comm_stream));
    }
  }
  VX_NCCL(ncclGroupEnd());
  return VX_OK;
}

// Emulated slabs: ghost planes <- neighbouring slabs' owned planes (device copies)
vx_status halo_local(vx_lattice* h) {
  for (size_t q = 0; q < h->slabs.size(); ++q) {
    const Slab& s = h->slabs[q];
    Arr mine[4];
    state_arrays(h, s, mine);
    for (int side = 0; side < 2; ++side) {
      const int nb = side == 0 ? (int)q - 1 : (int)q + 1;
      if (nb < 0 || nb >= (int)h->slabs.size()) continue;
      const Slab& o = h->slabs[nb];
      Arr theirs[4];
      state_arrays(h, o, theirs);
      const int x = side == 0 ? s.x0 - 1 : s.x1;   // ghost plane = neighbour's owned plane
      for (int a = 0; a < 4; ++a)
        VX_CUDA(cudaMemcpyAsync(plane_ptr(mine[a], s, x, h->plane), plane_ptr(theirs[a], o, x, h->plane),
                                h->plane * mine[a].esz, cudaMemcpyDeviceToDevice, h->stream));
    }
  }
  return VX_OK;
}

template <class R> vx_status enqueue_step(vx_lattice* h, cudaEvent_t* ev) {
  const bool col = h->collide();
  if (ev) VX_CUDA(cudaEventRecordWithFlags(ev[0], h->stream, cudaEventRecordExternal));
  ClockArgs ca{h->clk.as<Clock>(), h->dt, h->env.T_amp, h->env.T_freq, h->env.T_phase,
               0.5 * h->env.horizon_voxels * h->l, h->alpha_lo, h->alpha_hi, col ? 1 : 0,
               h->prec};
  if (col && h->nccl()) {
    // motion budget over the whole lattice: max |V| of every rank
    unsigned long long* vb = &h->clk.as<Clock>()->vmax_bits;
    VX_NCCL(ncclAllReduce(vb, vb, 1, ncclUint64, ncclMax, h->comm, h->stream));
  }
  k_clock<<<1, 32, 0, h->stream>>>(ca);
  if (col) {
    using R4 = typename VT<R>::R4;
    R4* ss = h->ss.as<R4>();
    const unsigned* gb = h->surf_d.as<unsigned>();
    // each slab's segment of the table was written by the previous step's update
    // (surface_entry) or by pack_surface after a state change
    if (h->nccl()) {   // every rank's segment of the surface table to every rank
      VX_NCCL(ncclGroupStart());
      for (int r = 0; r < h->nranks; ++r) {
        const size_t cnt = (size_t)(h->seg[r + 1] - h->seg[r]) * 2 * sizeof(R4);
        if (!cnt) continue;
        char* p = reinterpret_cast<char*>(ss + 2 * (size_t)h->seg[r]);
        VX_NCCL(ncclBroadcast(p, p, cnt, ncclInt8, r, h->comm, h->stream));
      }
      VX_NCCL(ncclGroupEnd());
    }
    const int S = (int)h->surf_g.size();
    BroadArgs b{gb, S, h->rows_begin(), h->rows_end(), h->cellh.as<int4>(),
                h->bcount.as<int>(), h->bstart.as<int>(), h->bitems.as<int>(),
                h->rowptr.as<int>(), h->col.as<int>(), h->cap, h->H, h->clk.as<Clock>(),
                h->batch_stride, h->batch_stride_z, h->batch_stride_y, h->sijk.as<int4>()};
    const double hc = h->cutoff * 1.001;
    {   // cooperative: all CTAs resident (grid-wide barriers between the phases)
      Dev<R> d0 = make_dev<R>(h, h->slabs[0]);
      double ox = h->origin[0], oy = h->origin[1], oz = h->origin[2];
      R hr = (R)hc, c2 = (R)(h->cutoff * h->cutoff);
      const R4* ssc = ss;
      void* args[] = {&d0, &b, &ssc, &ox, &oy, &oz, &hr, &c2};
      VX_CUDA(cudaLaunchCooperativeKernel((const void*)k_broadphase<R>, dim3(h->bp_grid), dim3(1024), args,
                                          0, h->stream));
    }
    for (size_t q = 0; q < h->slabs.size(); ++q) {
      const int s0 = h->slab_seg(q, 0), s1 = h->slab_seg(q, 1);
      if (s1 > s0)
        k_contact<R><<<grid_of((long long)(s1 - s0) * CONTACT_LANES), 256, 0, h->stream>>>(
            make_dev<R>(h, h->slabs[q]), gb, h->sijk.as<int4>(), ss, s0, s1,
                                                               h->rowptr.as<int>(), h->col.as<int>(),
                                                               (R)h->env.zeta_col);
    }
  }
  if (h->emulated) VX_TRY(halo_local(h));
  // (the fused engine has no bond-kernel interval: ev[1] would sit next to ev[2])
  if (ev && !h->fused()) VX_CUDA(cudaEventRecordWithFlags(ev[1], h->stream, cudaEventRecordExternal));
  if (h->fused()) {
    if (h->nccl()) {
      // ghost planes of S_n on the comm stream, overlapped with the interior
      // planes [x0+1, x1-1) (they read no ghost plane) on the main stream; the
      // two boundary planes follow the exchange on the comm stream, concurrently
      // with the interior pass
      const Slab& s = h->slabs[0];
      VX_CUDA(cudaEventRecord(h->ev_k4, h->stream));
      VX_CUDA(cudaStreamWaitEvent(h->comm_stream, h->ev_k4, 0));
      VX_TRY(halo_nccl(h));
      if (ev) VX_CUDA(cudaEventRecordWithFlags(ev[2], h->stream, cudaEventRecordExternal));
      VX_TRY(launch_fused<R>(h, s, col, s.x0 + 1, s.x1 - 1));
      VX_TRY(launch_boundary<R>(h, s, col, h->comm_stream));
      VX_CUDA(cudaEventRecord(h->ev_halo, h->comm_stream));
      VX_CUDA(cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
    } else {
      if (ev) VX_CUDA(cudaEventRecordWithFlags(ev[2], h->stream, cudaEventRecordExternal));
      for (const Slab& s : h->slabs) {
        if (h->emulated) {   // the launch split of the NCCL ranks (ghosts already copied)
          VX_TRY(launch_fused<R>(h, s, col, s.x0 + 1, s.x1 - 1));
          VX_TRY(launch_boundary<R>(h, s, col, h->stream));
        } else {
          VX_TRY(launch_fused<R>(h, s, col, s.x0, s.x1));
        }
      }
    }
    if (ev) VX_CUDA(cudaEventRecordWithFlags(ev[3], h->stream, cudaEventRecordExternal));
    VX_CUDA(cudaGetLastError());
    h->flip();
    return VX_OK;
  }
  if (h->nccl()) {
    // halo of S_n on the comm stream, overlapped with the interior bonds
    const Slab& s = h->slabs[0];
    const Dev<R> d = make_dev<R>(h, s);
    VX_CUDA(cudaEventRecord(h->ev_k4, h->stream));
    VX_CUDA(cudaStreamWaitEvent(h->comm_stream, h->ev_k4, 0));
    VX_TRY(halo_nccl(h));
    VX_CUDA(cudaEventRecord(h->ev_halo, h->comm_stream));
    launch_bonds<R>(h, s, d, s.x0, s.x1 - 1);
    VX_CUDA(cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
    launch_bonds<R>(h, s, d, s.xl0, s.x0);
    launch_bonds<R>(h, s, d, s.x1 - 1, s.x1);
  } else {
    for (const Slab& s : h->slabs) launch_bonds<R>(h, s, make_dev<R>(h, s), s.xl0, s.x1);
  }
  if (ev) VX_CUDA(cudaEventRecordWithFlags(ev[2], h->stream, cudaEventRecordExternal));
  for (const Slab& s : h->slabs) launch_integrate<R>(h, s, make_dev<R>(h, s), col);
  if (ev) VX_CUDA(cudaEventRecordWithFlags(ev[3], h->stream, cudaEventRecordExternal));
  VX_CUDA(cudaGetLastError());
  return VX_OK;
}

template <class R> vx_status pack_surface(vx_lattice* h) {
  using R4 = typename VT<R>::R4;
  for (size_t q = 0; q < h->slabs.size(); ++q) {
    const int s0 = h->slab_seg(q, 0), s1 = h->slab_seg(q, 1);
    if (s1 > s0)
      k_surf_pack<R><<<grid_of(s1 - s0), 256, 0, h->stream>>>(make_dev<R>(h, h->slabs[q]),
                                                               h->surf_d.as<unsigned>(), s0, s1,
                                                               h->ss.as<R4>());
  }
  VX_CUDA(cudaGetLastError());
  h->ss_dirty = false;
  return VX_OK;
}

// Accumulate the event times of one instrumented graph chunk (events of the
// measured steps only; pool offset `base`).
vx_status read_chunk_times(vx_lattice* h, size_t base, long long g) {
  for (long long s = 0; s < g; s += h->instr_stride) {
    cudaEvent_t* e = &h->events[base + (size_t)s * 4];
    VX_CUDA(cudaEventSynchronize(e[3]));
    float a = 0, b, c, t;
    if (h->fused()) {
      VX_CUDA(cudaEventElapsedTime(&c, e[0], e[2]));
    } else {
      VX_CUDA(cudaEventElapsedTime(&a, e[1], e[2]));
      VX_CUDA(cudaEventElapsedTime(&c, e[0], e[1]));
    }
    VX_CUDA(cudaEventElapsedTime(&b, e[2], e[3]));
    VX_CUDA(cudaEventElapsedTime(&t, e[0], e[3]));
    h->t_ms[0] += a; h->t_ms[1] += b; h->t_ms[2] += c; h->t_ms[3] += t;
    h->t_cnt[0] += h->fused() ? 0 : h->bond_launches();
    h->t_cnt[1] += h->fused() ? h->fused_launches() : (long long)h->slabs.size();
    h->t_cnt[2] += h->other_launches();
    h->t_cnt[3] += h->launches_per_step();
  }
  return VX_OK;
}

vx_status sync_state_copies(vx_lattice* h);

// VX_ENGINE_AUTO: pick the faster engine for this lattice once, at the first
// step.  Large lattices with full warps in z (nz >= 64, >= 4M cells) and
// slab-split lattices (every rank must pick the same engine, so no timing)
// take the fused engine unless a plane has < 32 cells (C5 1.24 vs 2.33 ms;
// shallow lattices run the (y, z)-mapped fused pass);
// otherwise both engines
// are timed as CUDA graphs of the same 8 steps' kernels -- the fused pass after
// its geometry tuning, the two-pass kernels on the spare state copy (K4 updates
// in place) -- and the faster one is kept.  Small lattices go either way: one
// C2 cube is faster fused (8.3 vs 11.4 us / step), 64 packed cubes or 4096
// packed cantilevers (nz = 20, 1) are faster two-pass (34 vs 39, 9 vs 44 us).
// Both engines produce the same S_{n+1}, so the choice only changes time.
template <class R> vx_status resolve_engine(vx_lattice* h) {
  Nvtx nvtx_("vx resolve engine");
  if (h->engine_req != VX_ENGINE_AUTO || h->engine_resolved) return VX_OK;
  h->engine_resolved = true;
  h->clear_graphs();
  if (h->emulated || h->nccl() || (h->nz >= 64 && h->nbox >= (1LL << 22))) {
    h->engine = (long long)h->ny * h->nz >= 32 ? VX_ENGINE_FUSED : VX_ENGINE_TWO_PASS;
    return prepare(h);   // bond records of the two-pass engine
  }
  const bool col = h->collide();
  Clock saved;
  VX_CUDA(cudaMemcpy(&saved, h->clk.p, sizeof saved, cudaMemcpyDeviceToHost));
  struct Ev {
    cudaEvent_t e = nullptr;
    ~Ev() { if (e) cudaEventDestroy(e); }
  } ev0, ev1;
  VX_CUDA(cudaEventCreate(&ev0.e));
  VX_CUDA(cudaEventCreate(&ev1.e));
  // 8 steps' kernels as one graph, launched once warm and 4 times timed
  auto time_graph = [&](auto&& body, float* ms) -> vx_status {
    cudaGraph_t g;
    VX_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    vx_status st = VX_OK;
    for (int r = 0; r < 8 && st == VX_OK; ++r) st = body();
    const cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
    if (st != VX_OK) return st;
    if (ce != cudaSuccess) return fail(VX_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t ex;
    const cudaError_t ie = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return fail(VX_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    cudaError_t se = cudaGraphLaunch(ex, h->stream);
    if (se == cudaSuccess) se = cudaEventRecord(ev0.e, h->stream);
    for (int r = 0; r < 4 && se == cudaSuccess; ++r) se = cudaGraphLaunch(ex, h->stream);
    if (se == cudaSuccess) se = cudaEventRecord(ev1.e, h->stream);
    if (se == cudaSuccess) se = cudaEventSynchronize(ev1.e);
    cudaGraphExecDestroy(ex);
    if (se != cudaSuccess) return fail(VX_ERR_CUDA, std::string("engine timing: ") + cudaGetErrorString(se));
    VX_CUDA(cudaEventElapsedTime(ms, ev0.e, ev1.e));
    return VX_OK;
  };
  float t_fused = 0, t_two = 0;
  h->engine = VX_ENGINE_FUSED;
  VX_TRY(tune_fused<R>(h));
  VX_TRY(time_graph([&]() -> vx_status {
    for (const Slab& s : h->slabs) VX_TRY(launch_fused<R>(h, s, col, s.x0, s.x1));
    return VX_OK;
  }, &t_fused));
  h->engine = VX_ENGINE_TWO_PASS;
  VX_TRY(prepare(h));   // bond records
  VX_TRY(sync_state_copies(h));
  h->flip();
  const vx_status st2 = time_graph([&]() -> vx_status {
    for (const Slab& s : h->slabs) launch_bonds<R>(h, s, make_dev<R>(h, s), s.xl0, s.x1);
    for (const Slab& s : h->slabs) launch_integrate<R>(h, s, make_dev<R>(h, s), col);
    return VX_OK;
  }, &t_two);
  h->flip();
  VX_TRY(st2);
  VX_TRY(sync_state_copies(h));   // the spare copy back to S_n
  VX_CUDA(cudaMemcpy(h->clk.p, &saved, sizeof saved, cudaMemcpyHostToDevice));
  h->ss_dirty = true;
  h->engine = t_two < t_fused ? VX_ENGINE_TWO_PASS : VX_ENGINE_FUSED;
  if (h->fused())
    for (Slab& s : h->slabs) { s.recA.release(); s.recB.release(); s.recC.release(); }
  if (std::getenv("VX_FUSED_TUNE_LOG"))
    std::fprintf(stderr, "voxsim: engine auto: fused %.2f us, two-pass %.2f us per step -> %s\n",
                 1e3 * t_fused / 32, 1e3 * t_two / 32, h->fused() ? "fused" : "two_pass");
  h->clear_graphs();
  return VX_OK;
}

// CUDA graphs of G steps; the remainder is captured as its own graph.  The
// fused engine ping-pongs two state copies, so a graph also depends on which
// copy is current when it starts (key = 2 g + parity).  With instrumentation
// on, the graphs carry event-record nodes around every launch class of every
// instr_stride-th step (their own cache); two event pools alternate between
// graph replays, so a chunk's times are read while the next chunk runs.
constexpr long long kGraphSteps = 32;

// The graph of g steps starting at state-copy parity `par`, event pool `pool`
// (captured and instantiated on first use).
template <class R>
vx_status get_graph(vx_lattice* h, long long g, int par, int pool, cudaGraphExec_t* out) {
  const long long G = kGraphSteps;
  const long long key = 2 * g + (h->fused() ? par : 0) +
                        (h->instr ? ((long long)h->instr_stride << 40) + ((long long)pool << 39) : 0);
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    const int par0 = h->slabs[0].par;
    for (auto& s : h->slabs) s.par = par;
    cudaGraph_t graph;
    VX_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    vx_status st = VX_OK;
    for (long long s = 0; s < g && st == VX_OK; ++s) {
      cudaEvent_t* ev = nullptr;
      if (h->instr && s % h->instr_stride == 0) ev = &h->events[(size_t)pool * G * 4 + (size_t)s * 4];
      st = enqueue_step<R>(h, ev);
    }
    cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
    for (auto& s : h->slabs) s.par = par0;   // capture only recorded the flips
    if (st != VX_OK) return st;
    if (ce != cudaSuccess) return fail(VX_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t ex;
    VX_CUDA(cudaGraphInstantiate(&ex, graph, 0));
    cudaGraphDestroy(graph);
    VX_CUDA(cudaGraphUpload(ex, h->stream));
    it = h->graphs.emplace(key, ex).first;
  }
  *out = it->second;
  return VX_OK;
}

// Everything a run of n steps needs before its first launch: the engine, the
// launch geometry, the surface table, the event pools.
template <class R> vx_status ready_steps(vx_lattice* h) {
  VX_TRY(resolve_engine<R>(h));
  VX_TRY(tune_fused<R>(h));
  if (h->collide() && h->ss_dirty) VX_TRY(pack_surface<R>(h));
  if (h->instr) {
    while (h->events.size() < (size_t)kGraphSteps * 8) {
      cudaEvent_t e;
      VX_CUDA(cudaEventCreate(&e));
      h->events.push_back(e);
    }
  }
  return VX_OK;
}

// The graphs vx_step(n) will replay, built without running them.
template <class R> vx_status prepare_graphs(vx_lattice* h, long long n) {
  VX_TRY(ready_steps<R>(h));
  long long left = n;
  int pool = 0, par = h->slabs[0].par;
  while (left > 0) {
    const long long g = left >= kGraphSteps ? kGraphSteps : left;
    cudaGraphExec_t ex;
    VX_TRY(get_graph<R>(h, g, par, pool, &ex));
    if (h->fused() && (g & 1)) par ^= 1;
    left -= g;
    if (h->instr) pool ^= 1;
  }
  VX_CUDA(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

template <class R> vx_status run_steps(vx_lattice* h, long long n) {
  VX_TRY(ready_steps<R>(h));
  const long long G = kGraphSteps;
  long long left = n;
  int pool = 0;
  long long pending = 0;   // steps of the chunk in flight whose times are unread
  while (left > 0) {
    const long long g = left >= G ? G : left;
    cudaGraphExec_t ex;
    VX_TRY(get_graph<R>(h, g, h->slabs[0].par, pool, &ex));
    Nvtx r_(h->fused() ? "vx steps graph (fused)" : "vx steps graph (two-pass)");
    VX_CUDA(cudaGraphLaunch(ex, h->stream));
    if (h->fused() && (g & 1)) h->flip();
    left -= g;
    if (h->instr) {
      if (pending) VX_TRY(read_chunk_times(h, (size_t)(pool ^ 1) * G * 4, pending));
      pending = g;
      pool ^= 1;
    }
  }
  if (h->instr && pending) VX_TRY(read_chunk_times(h, (size_t)(pool ^ 1) * G * 4, pending));
  VX_CUDA(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

vx_status check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(VX_ERR_NO_DEVICE, "no CUDA device visible (no CPU fallback)");
  }
  return VX_OK;
}

vx_status set_device(const vx_lattice* h) {
  VX_CUDA(cudaSetDevice(h->device));
  return VX_OK;
}

// Copy the current state into the fused engine's second buffer (allocated on
// first use); needed before fused steps after any host-side state change.
vx_status sync_state_copies(vx_lattice* h) {
  for (Slab& s : h->slabs)
    for (int a = 0; a < 4; ++a) {
      const DevBuf& c = s.buf[s.par][a];
      DevBuf& o = s.buf[s.par ^ 1][a];
      VX_TRY(o.alloc(c.bytes));
      VX_CUDA(cudaMemcpyAsync(o.p, c.p, c.bytes, cudaMemcpyDeviceToDevice, h->stream));
    }
  VX_CUDA(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

vx_status set_force_rebuild(vx_lattice* h) {
  Clock* c = h->clk.as<Clock>();
  int one = 1;
  VX_CUDA(cudaMemcpy(&c->force_rebuild, &one, 4, cudaMemcpyHostToDevice));
  return VX_OK;
}

// Owned planes -> box-ordered fp64 SoA (14 components x nbox) on every rank.
vx_status read_box(vx_lattice* h, double* boxbuf) {
  for (const Slab& s : h->slabs) {
    const uint32_t beg = (uint32_t)(s.x0 - s.xl0) * h->plane, end = (uint32_t)(s.x1 - s.xl0) * h->plane;
    if (h->prec == 32)
      k_pack_box<float><<<grid_of(end - beg), 256, 0, h->stream>>>(make_dev<float>(h, s), beg, end, s.box_base,
                                                                   h->nbox, boxbuf, h->origin[0], h->origin[1], h->origin[2]);
    else
      k_pack_box<double><<<grid_of(end - beg), 256, 0, h->stream>>>(make_dev<double>(h, s), beg, end, s.box_base,
                                                                    h->nbox, boxbuf, h->origin[0], h->origin[1], h->origin[2]);
    VX_CUDA(cudaGetLastError());
  }
  if (h->nccl()) {
    VX_NCCL(ncclGroupStart());
    for (int r = 0; r < h->nranks; ++r) {
      int x0, x1;
      slab_planes(h->nx, h->nranks, r, &x0, &x1);
      const size_t cnt = (size_t)(x1 - x0) * h->plane;
      for (int c = 0; c < 14; ++c) {
        double* p = boxbuf + (size_t)c * h->nbox + (size_t)x0 * h->plane;
        VX_NCCL(ncclBroadcast(p, p, cnt, ncclDouble, r, h->comm, h->stream));
      }
    }
    VX_NCCL(ncclGroupEnd());
  }
  return VX_OK;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

const char* vx_last_error(void) { return g_err.c_str(); }
int32_t vx_abi_version(void) { return VOXSIM_ABI_VERSION; }

vx_status vx_slab_planes(int32_t nx, int32_t nranks, int32_t rank, int32_t* x_begin, int32_t* x_end) {
  if (nx < 1 || nranks < 1 || nranks > nx || rank < 0 || rank >= nranks || !x_begin || !x_end)
    return fail(VX_ERR_INVALID_ARG, "bad slab arguments");
  slab_planes(nx, nranks, rank, x_begin, x_end);
  return VX_OK;
}

vx_status vx_nccl_unique_id(void* out128) {
  if (!out128) return fail(VX_ERR_INVALID_ARG, "out128 is NULL");
  ncclUniqueId id;
  VX_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
  return VX_OK;
}

vx_status vx_create_lattice(const vx_lattice_desc* desc, vx_lattice** out) {
  Nvtx nvtx_("vx_create_lattice");
  if (!out) return fail(VX_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!desc || !desc->cells) return fail(VX_ERR_INVALID_ARG, "desc or desc->cells is NULL");
  if (desc->nx < 1 || desc->ny < 1 || desc->nz < 1)
    return fail(VX_ERR_INVALID_ARG, "nx, ny, nz must be >= 1");
  if (!(desc->lattice_dim > 0) || !std::isfinite(desc->lattice_dim))
    return fail(VX_ERR_INVALID_ARG, "lattice_dim must be > 0");
  if (desc->precision != 32 && desc->precision != 64)
    return fail(VX_ERR_INVALID_ARG, "precision must be 32 or 64");
  if (desc->nranks < 1 || desc->rank < 0 || desc->rank >= desc->nranks)
    return fail(VX_ERR_INVALID_ARG, "bad rank / nranks");
  if (desc->nranks > desc->nx) return fail(VX_ERR_INVALID_ARG, "nranks > nx (empty slab)");
  const bool emulated = desc->nranks > 1 && !desc->nccl_id;
  if (emulated && desc->rank != 0)
    return fail(VX_ERR_INVALID_ARG, "emulated slabs (nccl_id NULL) need rank 0");
  const long long cells = (long long)desc->nx * desc->ny * desc->nz;
  if (cells >= (1LL << 32)) return fail(VX_ERR_INVALID_ARG, "workspace too large (>= 2^32 cells)");
  VX_TRY(check_device());
  vx_lattice* h = new vx_lattice();
  h->nx = desc->nx; h->ny = desc->ny; h->nz = desc->nz;
  h->l = desc->lattice_dim;
  for (int c = 0; c < 3; ++c) h->origin[c] = desc->origin[c];
  h->prec = desc->precision;
  h->device = desc->device; h->rank = desc->rank; h->nranks = desc->nranks;
  h->emulated = emulated;
  // one rank with a unique id and VX_FORCE_NCCL=1: every NCCL call of the slab
  // path runs (an empty ghost exchange, one-rank broadcasts / reductions), so a
  // single GPU exercises the multi-rank code: communicator, comm-stream overlap,
  // NCCL inside CUDA graphs
  if (desc->nranks == 1 && desc->nccl_id && std::getenv("VX_FORCE_NCCL")) h->force_nccl = true;
  if (const char* e = std::getenv("VX_FUSED_YZ")) h->yz_ok = std::atoi(e) != 0;
  if (const char* e = std::getenv("VX_FUSED_TY")) {
    h->fused_ty = std::max(1, std::min(64, std::atoi(e)));
    h->fused_tune = 0;   // an explicit geometry is not tuned away
  }
  if (const char* e = std::getenv("VX_FUSED_WAVES")) {
    h->fused_waves = std::max(1, std::min(64, std::atoi(e)));
    h->fused_tune = 0;
  }
  if (const char* e = std::getenv("VX_FUSED_SX")) {   // planes per segment (experiments)
    h->fused_sx = std::max(1, std::min(512, std::atoi(e)));
    h->fused_tune = 0;
  }
  if (const char* e = std::getenv("VX_FUSED_TUNE")) h->fused_tune = std::atoi(e);
  h->cells.assign(desc->cells, desc->cells + cells);
  h->plane = (uint32_t)((long long)h->ny * h->nz);
  h->nbox = (long long)h->nx * h->plane;
  const int nslab = emulated ? h->nranks : 1;
  h->slabs.resize(nslab);
  for (int q = 0; q < nslab; ++q) {
    Slab& s = h->slabs[q];
    slab_planes(h->nx, h->nranks, emulated ? q : h->rank, &s.x0, &s.x1);
    s.xl0 = std::max(s.x0 - 1, 0);
    s.xl1 = std::min(s.x1 + 1, h->nx);
    s.nloc = (uint32_t)((long long)(s.xl1 - s.xl0) * h->plane);
    s.box_base = (long long)s.xl0 * h->plane;
  }
  h->x0 = h->slabs.front().x0;
  h->x1 = h->slabs.back().x1;
  auto bail = [&](vx_status s) { std::string m = g_err; vx_destroy(h); g_err = m; return s; };
  vx_status s = set_device(h);
  if (s != VX_OK) return bail(s);
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_k4, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(VX_ERR_CUDA, "stream/event creation failed"));
  if ((s = build_topology(h)) != VX_OK) return bail(s);
  const size_t r = rsize(h->prec);
  if ((s = h->clk.alloc(sizeof(Clock)))) return bail(s);
  for (Slab& sl : h->slabs) {
    const size_t n = sl.nloc;
    if ((s = sl.pos().alloc(n * 4 * r)) || (s = sl.quat().alloc(n * 4 * r)) || (s = sl.mom().alloc(n * 4 * r)) ||
        (s = sl.ang().alloc(n * 2 * r)) ||
        (s = sl.meta_d.alloc(n * 4)) || (s = sl.ext_of_local.alloc(n * 4)))
      return bail(s);
    // initial state: at rest on the lattice sites, identity orientation (.w = 1);
    // external id of every local box (0xffffffff: empty)
    cudaStream_t st = h->stream;
    if (cudaMemsetAsync(sl.pos().p, 0, sl.pos().bytes, st) != cudaSuccess ||
        cudaMemsetAsync(sl.mom().p, 0, sl.mom().bytes, st) != cudaSuccess ||
        cudaMemsetAsync(sl.ang().p, 0, sl.ang().bytes, st) != cudaSuccess ||
        cudaMemsetAsync(sl.ext_of_local.p, 0xff, n * 4, st) != cudaSuccess)
      return bail(fail(VX_ERR_CUDA, "memset failed"));
    if (r == 4)
      k_topo_quat_identity<float><<<grid_of((uint32_t)n), 256, 0, st>>>(sl.quat().as<float4>(), (uint32_t)n);
    else
      k_topo_quat_identity<double><<<grid_of((uint32_t)n), 256, 0, st>>>(sl.quat().as<double4>(), (uint32_t)n);
    if (h->N)
      k_topo_eol<<<topo_grid((unsigned long long)h->N), 256, 0, st>>>(h->box_of_ext_d.as<long long>(), h->N,
                                                                      sl.box_base, (uint32_t)n,
                                                                      sl.ext_of_local.as<uint32_t>());
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
      return bail(fail(VX_ERR_CUDA, "state initialisation failed"));
  }
  if ((s = sync_state_copies(h)) != VX_OK) return bail(s);
  Clock c0{};
  c0.err = ~0ULL;
  c0.fault = ~0ULL;
  c0.force_rebuild = 1;
  if (cudaMemcpy(h->clk.p, &c0, sizeof c0, cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(fail(VX_ERR_CUDA, "upload failed"));
  h->fixed.assign((size_t)h->N, 0);
  h->fext.assign((size_t)h->N * 3, 0.0);
  if ((s = upload_meta(h)) != VX_OK) return bail(s);
  if (h->nccl()) {
    ncclUniqueId id;
    std::memcpy(&id, desc->nccl_id, sizeof id);
    ncclResult_t nr = ncclCommInitRank(&h->comm, h->nranks, id, h->rank);
    if (nr != ncclSuccess) return bail(fail(VX_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(nr)));
  }
  *out = h;
  return VX_OK;
}

void vx_destroy(vx_lattice* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->clear_graphs();
  for (auto e : h->events) cudaEventDestroy(e);
  if (h->comm) ncclCommDestroy(h->comm);
  if (h->ev_k4) cudaEventDestroy(h->ev_k4);
  if (h->ev_halo) cudaEventDestroy(h->ev_halo);
  if (h->stream) cudaStreamDestroy(h->stream);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  delete h;
}

vx_status vx_set_materials(vx_lattice* h, const vx_material* p, int32_t n) {
  if (!h || !p || n < 1 || n > 255) return fail(VX_ERR_INVALID_ARG, "bad palette (need 1..255 materials)");
  for (int i = 0; i < n; ++i) {
    const vx_material& m = p[i];
    if (!(m.E > 0) || !(m.rho > 0) || !(m.nu > -1 && m.nu < 0.5) || !(m.mu_d >= 0) ||
        !(m.mu_s >= m.mu_d) || !std::isfinite(m.E) || !std::isfinite(m.rho) || !std::isfinite(m.cte))
      return fail(VX_ERR_INVALID_ARG, "material " + std::to_string(i) +
                                          " violates E>0, rho>0, -1<nu<0.5, mu_s>=mu_d>=0");
  }
  if (h->max_cell > n)
    return fail(VX_ERR_OUT_OF_RANGE, "a cell references material " + std::to_string(h->max_cell) +
                                         " of a " + std::to_string(n) + "-entry palette");
  VX_TRY(set_device(h));
  h->mats.assign(p, p + n);
  if (h->prec == 32) VX_TRY(compute_dt<float>(h));
  else VX_TRY(compute_dt<double>(h));
  h->mats_set = true;
  h->tables_dirty = true;
  VX_TRY(set_force_rebuild(h));
  update_dt(h);
  return VX_OK;
}

vx_status vx_set_environment(vx_lattice* h, const vx_env* e) {
  if (!h || !e) return fail(VX_ERR_INVALID_ARG, "NULL argument");
  auto ratio_ok = [](double z) { return z >= 0 && z <= 1; };
  if (!ratio_ok(e->zeta_bond) || !ratio_ok(e->zeta_ground) || !ratio_ok(e->zeta_col))
    return fail(VX_ERR_INVALID_ARG, "damping ratios must lie in [0,1] (App. B)");
  if (!(e->dt_safety > 0 && e->dt_safety <= 1)) return fail(VX_ERR_INVALID_ARG, "dt_safety must be in (0,1]");
  if (e->self_collision && !(e->horizon_voxels > 0))
    return fail(VX_ERR_INVALID_ARG, "horizon_voxels must be > 0");
  const double v[] = {e->gravity, e->floor_z, e->T_ref, e->T_amp, e->T_freq, e->T_phase};
  for (double x : v)
    if (!std::isfinite(x)) return fail(VX_ERR_INVALID_ARG, "non-finite environment value");
  VX_TRY(set_device(h));
  h->env = *e;
  h->env_set = true;
  h->tables_dirty = true;
  update_dt(h);
  VX_TRY(set_force_rebuild(h));
  h->clear_graphs();
  return VX_OK;
}

vx_status vx_set_boundary(vx_lattice* h, const uint8_t* fixed, const double* f_ext) {
  if (!h) return fail(VX_ERR_INVALID_ARG, "NULL handle");
  VX_TRY(set_device(h));
  std::vector<double> fe((size_t)h->N * 3, 0.0);
  bool any = false;
  if (f_ext)
    for (long long i = 0; i < 3 * h->N; ++i) {
      if (!std::isfinite(f_ext[i])) return fail(VX_ERR_INVALID_ARG, "non-finite external force");
      fe[i] = f_ext[i];
      any |= f_ext[i] != 0;
    }
  h->fixed.assign((size_t)h->N, 0);
  if (fixed) std::copy(fixed, fixed + h->N, h->fixed.begin());
  h->fext.swap(fe);
  h->any_ext = any;
  return upload_meta(h);
}

vx_status vx_add_region(vx_lattice* h, int32_t kind, const double o[3], const double sz[3],
                        const double force[3]) {
  if (!h || !o || !sz) return fail(VX_ERR_INVALID_ARG, "NULL argument");
  if (kind != 0 && kind != 1) return fail(VX_ERR_INVALID_ARG, "kind must be 0 (fixed) or 1 (forced)");
  if (kind == 1 && !force) return fail(VX_ERR_INVALID_ARG, "forced region needs a force");
  for (int d = 0; d < 3; ++d)
    if (!(o[d] >= 0 && o[d] <= 1 && sz[d] >= 0 && o[d] + sz[d] <= 1 + 1e-12))
      return fail(VX_ERR_INVALID_ARG, "region must lie within the workspace fractions [0,1]");
  VX_TRY(set_device(h));
  const int dims[3] = {h->nx, h->ny, h->nz};
  std::vector<long long> hit;
  for (long long e = 0; e < h->N; ++e) {
    const long long g = h->box_of_ext[e];
    const long long idx[3] = {g / h->plane, (g / h->nz) % h->ny, g % h->nz};
    bool in = true;
    for (int d = 0; d < 3 && in; ++d) {
      const double lo = o[d] * dims[d], hi = (o[d] + sz[d]) * dims[d];
      const double c0 = (double)idx[d], c1 = c0 + 1.0;
      in = (hi > lo) ? (std::max(lo, c0) < std::min(hi, c1)) : (c0 <= lo && lo <= c1);
    }
    if (in) hit.push_back(e);
  }
  if (kind == 0) {
    for (long long e : hit) h->fixed[e] = 1;
  } else if (!hit.empty()) {
    const double inv = 1.0 / (double)hit.size();
    for (long long e : hit)
      for (int c = 0; c < 3; ++c) {
        h->fext[3 * e + c] += force[c] * inv;
        h->any_ext |= h->fext[3 * e + c] != 0;
      }
  }
  return upload_meta(h);
}

vx_status vx_set_state(vx_lattice* h, const double* pos, const double* quat, const double* lin,
                       const double* ang, const uint8_t* latch) {
  Nvtx nvtx_("vx_set_state");
  if (!h) return fail(VX_ERR_INVALID_ARG, "NULL handle");
  VX_TRY(set_device(h));
  const long long N = h->N;
  if (N == 0) return VX_OK;
  DevBuf& b = h->stage_ext;   // kept: state I/O every episode must not pay cudaMalloc / cudaFree
  const size_t off[5] = {0, (size_t)N * 3, (size_t)N * 7, (size_t)N * 10, (size_t)N * 13};
  VX_TRY(b.alloc((size_t)N * 13 * 8 + (size_t)N));
  double* bd = b.as<double>();
  uint8_t* bl = reinterpret_cast<uint8_t*>(bd + off[4]);
  if (pos) VX_CUDA(cudaMemcpyAsync(bd + off[0], pos, (size_t)N * 24, cudaMemcpyHostToDevice, h->stream));
  if (quat) VX_CUDA(cudaMemcpyAsync(bd + off[1], quat, (size_t)N * 32, cudaMemcpyHostToDevice, h->stream));
  if (lin) VX_CUDA(cudaMemcpyAsync(bd + off[2], lin, (size_t)N * 24, cudaMemcpyHostToDevice, h->stream));
  if (ang) VX_CUDA(cudaMemcpyAsync(bd + off[3], ang, (size_t)N * 24, cudaMemcpyHostToDevice, h->stream));
  if (latch) VX_CUDA(cudaMemcpyAsync(bl, latch, (size_t)N, cudaMemcpyHostToDevice, h->stream));
  const long long* boe = h->box_of_ext_d.as<long long>();
  for (const Slab& s : h->slabs) {   // owned and ghost planes alike
    if (h->prec == 32)
      k_scatter_state<float><<<grid_of(N), 256, 0, h->stream>>>(
          make_dev<float>(h, s), boe, N, s.box_base, pos ? bd + off[0] : nullptr, quat ? bd + off[1] : nullptr,
          lin ? bd + off[2] : nullptr, ang ? bd + off[3] : nullptr, latch ? bl : nullptr, h->origin[0],
          h->origin[1], h->origin[2]);
    else
      k_scatter_state<double><<<grid_of(N), 256, 0, h->stream>>>(
          make_dev<double>(h, s), boe, N, s.box_base, pos ? bd + off[0] : nullptr, quat ? bd + off[1] : nullptr,
          lin ? bd + off[2] : nullptr, ang ? bd + off[3] : nullptr, latch ? bl : nullptr, h->origin[0],
          h->origin[1], h->origin[2]);
    VX_CUDA(cudaGetLastError());
  }
  VX_CUDA(cudaStreamSynchronize(h->stream));
  h->ss_dirty = true;
  return set_force_rebuild(h);
}

namespace {
struct CkptHeader {
  uint64_t magic;
  int32_t prec, rank;
  int64_t nloc, N, steps_done;
};
const uint64_t kCkptMagic = 0x32504b43584f56ULL;  // "VOXCKP2"
int64_t ckpt_nloc(const vx_lattice* h) {
  int64_t n = 0;
  for (const Slab& s : h->slabs) n += s.nloc;
  return n;
}
}  // namespace

int64_t vx_checkpoint_bytes(const vx_lattice* h) {
  if (!h) return -1;
  int64_t b = sizeof(CkptHeader) + sizeof(Clock);
  for (const Slab& s : h->slabs) b += (int64_t)(s.pos().bytes + s.quat().bytes + s.mom().bytes + s.ang().bytes);
  return b;
}

vx_status vx_save_checkpoint(vx_lattice* h, void* buf, int64_t bytes) {
  Nvtx nvtx_("vx_save_checkpoint");
  if (!h || !buf || bytes < vx_checkpoint_bytes(h)) return fail(VX_ERR_INVALID_ARG, "bad checkpoint buffer");
  VX_TRY(set_device(h));
  char* p = static_cast<char*>(buf);
  CkptHeader hd{kCkptMagic, h->prec, h->rank, ckpt_nloc(h), h->N, h->steps_done};
  std::memcpy(p, &hd, sizeof hd);
  p += sizeof hd;
  for (Slab& s : h->slabs)
    for (DevBuf* b : {&s.pos(), &s.quat(), &s.mom(), &s.ang()}) {
      VX_CUDA(cudaMemcpy(p, b->p, b->bytes, cudaMemcpyDeviceToHost));
      p += b->bytes;
    }
  VX_CUDA(cudaMemcpy(p, h->clk.p, sizeof(Clock), cudaMemcpyDeviceToHost));
  return VX_OK;
}

vx_status vx_load_checkpoint(vx_lattice* h, const void* buf, int64_t bytes) {
  Nvtx nvtx_("vx_load_checkpoint");
  if (!h || !buf || bytes < vx_checkpoint_bytes(h)) return fail(VX_ERR_INVALID_ARG, "bad checkpoint buffer");
  VX_TRY(set_device(h));
  const char* p = static_cast<const char*>(buf);
  CkptHeader hd;
  std::memcpy(&hd, p, sizeof hd);
  if (hd.magic != kCkptMagic || hd.prec != h->prec || hd.nloc != ckpt_nloc(h) || hd.N != h->N ||
      hd.rank != h->rank)
    return fail(VX_ERR_INVALID_ARG, "checkpoint does not match this lattice (shape, precision or rank)");
  p += sizeof hd;
  for (Slab& s : h->slabs)
    for (DevBuf* b : {&s.pos(), &s.quat(), &s.mom(), &s.ang()}) {
      VX_CUDA(cudaMemcpy(b->p, p, b->bytes, cudaMemcpyHostToDevice));
      p += b->bytes;
    }
  Clock c;
  std::memcpy(&c, p, sizeof c);
  c.force_rebuild = 1;   // the pair list is rebuilt from the restored state
  c.err = ~0ULL;
  c.fault = ~0ULL;
  c.overflow = 0;
  VX_CUDA(cudaMemcpy(h->clk.p, &c, sizeof c, cudaMemcpyHostToDevice));
  h->steps_done = hd.steps_done;
  h->ss_dirty = true;
  // static meta bits follow this lattice's boundary conditions (latch kept)
  return upload_meta(h);
}

vx_status vx_set_step(vx_lattice* h, int64_t n) {
  if (!h || n < 0) return fail(VX_ERR_INVALID_ARG, "bad argument");
  VX_TRY(set_device(h));
  Clock* c = h->clk.as<Clock>();
  long long v = n;
  VX_CUDA(cudaMemcpy(&c->next, &v, 8, cudaMemcpyHostToDevice));
  h->steps_done = n;
  return VX_OK;
}

vx_status vx_prepare_steps(vx_lattice* h, int64_t n) {
  Nvtx nvtx_("vx_prepare_steps");
  if (!h || n < 0) return fail(VX_ERR_INVALID_ARG, "bad argument");
  if (n == 0) return VX_OK;
  VX_TRY(set_device(h));
  VX_TRY(prepare(h));
  if (h->N == 0) return VX_OK;
  if (h->prec == 32) return prepare_graphs<float>(h, n);
  return prepare_graphs<double>(h, n);
}

vx_status vx_step(vx_lattice* h, int64_t n) {
  Nvtx nvtx_("vx_step");
  if (!h || n < 0) return fail(VX_ERR_INVALID_ARG, "bad argument");
  if (n == 0) return VX_OK;
  VX_TRY(set_device(h));
  VX_TRY(prepare(h));
  if (h->N == 0) { h->steps_done += n; return VX_OK; }
  if (h->prec == 32) VX_TRY(run_steps<float>(h, n));
  else VX_TRY(run_steps<double>(h, n));
  h->steps_done += n;
#ifdef VX_CHECKED
  {   // device checks (vx_common.cuh): the first failure, as VX_ERR_STATE
    unsigned long long chk = 0;
    VX_CUDA(cudaMemcpyFromSymbol(&chk, vx::g_vx_chk, sizeof chk));
    if (chk) {
      static const char* what[] = {"?", "state load index out of range", "-z record race (k_step_fused)",
                                   "edge row race (k_step_fused)", "material index out of range",
                                   "-y ring race (k_step_fused_yz)", "-z record race (k_step_fused_yz)",
                                   "state store outside the launch's planes"};
      const unsigned code = (unsigned)(chk >> 32);
      return fail(VX_ERR_STATE, std::string("device check failed: ") + (code < 8 ? what[code] : "?") +
                                    " (code " + std::to_string(code) + ", kernel source line " +
                                    std::to_string((unsigned)(chk & 0xffffffffu)) + ")");
    }
  }
#endif
  Clock c;
  VX_CUDA(cudaMemcpy(&c, h->clk.p, sizeof c, cudaMemcpyDeviceToHost));
  unsigned long long err = c.err, fault = c.fault;
  int overflow = c.overflow;
  if (h->nccl()) {   // every rank returns the same status
    DevBuf t;
    VX_TRY(t.alloc(24));
    unsigned long long hv[3] = {err, fault, ~0ULL - (unsigned long long)overflow};
    VX_CUDA(cudaMemcpy(t.p, hv, 24, cudaMemcpyHostToDevice));
    VX_NCCL(ncclAllReduce(t.p, t.p, 3, ncclUint64, ncclMin, h->comm, h->stream));
    VX_CUDA(cudaMemcpyAsync(hv, t.p, 24, cudaMemcpyDeviceToHost, h->stream));
    VX_CUDA(cudaStreamSynchronize(h->stream));
    err = hv[0];
    fault = hv[1];
    overflow = (int)(~0ULL - hv[2]);
  }
  if (overflow) return fail(VX_ERR_STATE, "contact pair list capacity exceeded");
  if (fault != ~0ULL)
    return fail(VX_ERR_DIVERGED, "non-positive thermal rest length at step " + std::to_string(fault) + " (S:205)");
  if (err != ~0ULL) {
    const long long step = (long long)(err >> 32);
    const long long ext = (long long)(err & 0xffffffffULL);
    return fail(VX_ERR_DIVERGED, "diverged: voxel " + std::to_string(ext) + " at step " + std::to_string(step));
  }
  return VX_OK;
}

vx_status vx_read_state(vx_lattice* h, double* pos, double* quat, double* lin, double* ang,
                        uint8_t* latch) {
  Nvtx nvtx_("vx_read_state");
  if (!h) return fail(VX_ERR_INVALID_ARG, "NULL handle");
  VX_TRY(set_device(h));
  const long long N = h->N;
  if (N == 0) return VX_OK;
  DevBuf& box = h->stage_box;
  DevBuf& ext = h->stage_ext;
  VX_TRY(box.alloc((size_t)h->nbox * 14 * 8));
  VX_TRY(ext.alloc((size_t)N * 13 * 8 + (size_t)N));
  VX_TRY(read_box(h, box.as<double>()));
  double* e = ext.as<double>();
  uint8_t* el = reinterpret_cast<uint8_t*>(e + (size_t)N * 13);
  k_box_to_ext<<<grid_of(N), 256, 0, h->stream>>>(box.as<double>(), h->nbox, h->box_of_ext_d.as<long long>(), N,
                                                  e, e + (size_t)N * 3, e + (size_t)N * 7, e + (size_t)N * 10, el);
  VX_CUDA(cudaGetLastError());
  if (pos) VX_CUDA(cudaMemcpyAsync(pos, e, (size_t)N * 24, cudaMemcpyDeviceToHost, h->stream));
  if (quat) VX_CUDA(cudaMemcpyAsync(quat, e + (size_t)N * 3, (size_t)N * 32, cudaMemcpyDeviceToHost, h->stream));
  if (lin) VX_CUDA(cudaMemcpyAsync(lin, e + (size_t)N * 7, (size_t)N * 24, cudaMemcpyDeviceToHost, h->stream));
  if (ang) VX_CUDA(cudaMemcpyAsync(ang, e + (size_t)N * 10, (size_t)N * 24, cudaMemcpyDeviceToHost, h->stream));
  if (latch) VX_CUDA(cudaMemcpyAsync(latch, el, (size_t)N, cudaMemcpyDeviceToHost, h->stream));
  VX_CUDA(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

// The owned-voxel lists (vx_num_owned ...), built once.
static vx_status ensure_owned(vx_lattice* h) {
  if (h->owned_ready) return VX_OK;
  const long long lo = (long long)h->x0 * h->plane, hi = (long long)h->x1 * h->plane;
  h->owned_ext.clear();
  std::vector<long long> box;
  std::vector<std::vector<long long>> lid(h->slabs.size()), gid(h->slabs.size()), dst(h->slabs.size());
  for (long long e = 0; e < h->N; ++e) {
    const long long g = h->box_of_ext[e];
    if (g < lo || g >= hi) continue;
    const long long t = (long long)h->owned_ext.size();
    h->owned_ext.push_back(e);
    box.push_back(g);
    const long long x = g / h->plane;
    for (size_t q = 0; q < h->slabs.size(); ++q) {
      const Slab& s = h->slabs[q];
      if (x >= s.x0 && x < s.x1) {
        lid[q].push_back(g - s.box_base);
        gid[q].push_back(g);
        dst[q].push_back(t);
      }
    }
  }
  const size_t M = box.size();
  VX_TRY(h->owned_box_d.alloc(M * 8));
  if (M) VX_CUDA(cudaMemcpy(h->owned_box_d.p, box.data(), M * 8, cudaMemcpyHostToDevice));
  for (size_t q = 0; q < h->slabs.size(); ++q) {
    Slab& s = h->slabs[q];
    const size_t m = lid[q].size();
    s.own_n = (long long)m;
    VX_TRY(s.own_lid.alloc(m * 8));
    VX_TRY(s.own_gid.alloc(m * 8));
    VX_TRY(s.own_dst.alloc(m * 8));
    if (!m) continue;
    VX_CUDA(cudaMemcpy(s.own_lid.p, lid[q].data(), m * 8, cudaMemcpyHostToDevice));
    VX_CUDA(cudaMemcpy(s.own_gid.p, gid[q].data(), m * 8, cudaMemcpyHostToDevice));
    VX_CUDA(cudaMemcpy(s.own_dst.p, dst[q].data(), m * 8, cudaMemcpyHostToDevice));
  }
  h->owned_ready = true;
  return VX_OK;
}

int64_t vx_num_owned(const vx_lattice* h) {
  if (!h) return -1;
  if (vx_lattice* m = const_cast<vx_lattice*>(h); ensure_owned(m) != VX_OK) return -1;
  return (int64_t)h->owned_ext.size();
}

vx_status vx_owned_ids(const vx_lattice* h, int64_t* ids) {
  if (!h || !ids) return fail(VX_ERR_INVALID_ARG, "bad argument");
  VX_TRY(ensure_owned(const_cast<vx_lattice*>(h)));
  if (!h->owned_ext.empty()) std::memcpy(ids, h->owned_ext.data(), h->owned_ext.size() * 8);
  return VX_OK;
}

vx_status vx_set_state_owned(vx_lattice* h, const double* pos, const double* quat, const double* lin,
                             const double* ang, const uint8_t* latch) {
  Nvtx nvtx_("vx_set_state_owned");
  if (!h) return fail(VX_ERR_INVALID_ARG, "NULL handle");
  VX_TRY(set_device(h));
  VX_TRY(ensure_owned(h));
  const long long M = (long long)h->owned_ext.size();
  if (M == 0) return VX_OK;
  DevBuf& b = h->stage_ext;
  const size_t off[5] = {0, (size_t)M * 3, (size_t)M * 7, (size_t)M * 10, (size_t)M * 13};
  if (b.bytes < (size_t)M * 13 * 8 + (size_t)M) VX_TRY(b.alloc((size_t)M * 13 * 8 + (size_t)M));
  double* bd = b.as<double>();
  uint8_t* bl = reinterpret_cast<uint8_t*>(bd + off[4]);
  if (pos) VX_CUDA(cudaMemcpyAsync(bd + off[0], pos, (size_t)M * 24, cudaMemcpyHostToDevice, h->stream));
  if (quat) VX_CUDA(cudaMemcpyAsync(bd + off[1], quat, (size_t)M * 32, cudaMemcpyHostToDevice, h->stream));
  if (lin) VX_CUDA(cudaMemcpyAsync(bd + off[2], lin, (size_t)M * 24, cudaMemcpyHostToDevice, h->stream));
  if (ang) VX_CUDA(cudaMemcpyAsync(bd + off[3], ang, (size_t)M * 24, cudaMemcpyHostToDevice, h->stream));
  if (latch) VX_CUDA(cudaMemcpyAsync(bl, latch, (size_t)M, cudaMemcpyHostToDevice, h->stream));
  const long long* boe = h->owned_box_d.as<long long>();
  for (const Slab& s : h->slabs) {   // entry e goes to box owned_box[e] (any slab whose box holds it)
    if (h->prec == 32)
      k_scatter_state<float><<<grid_of(M), 256, 0, h->stream>>>(
          make_dev<float>(h, s), boe, M, s.box_base, pos ? bd + off[0] : nullptr, quat ? bd + off[1] : nullptr,
          lin ? bd + off[2] : nullptr, ang ? bd + off[3] : nullptr, latch ? bl : nullptr, h->origin[0],
          h->origin[1], h->origin[2]);
    else
      k_scatter_state<double><<<grid_of(M), 256, 0, h->stream>>>(
          make_dev<double>(h, s), boe, M, s.box_base, pos ? bd + off[0] : nullptr, quat ? bd + off[1] : nullptr,
          lin ? bd + off[2] : nullptr, ang ? bd + off[3] : nullptr, latch ? bl : nullptr, h->origin[0],
          h->origin[1], h->origin[2]);
    VX_CUDA(cudaGetLastError());
  }
  VX_CUDA(cudaStreamSynchronize(h->stream));
  h->ss_dirty = true;
  return set_force_rebuild(h);
}

vx_status vx_read_state_owned(vx_lattice* h, double* pos, double* quat, double* lin, double* ang,
                              uint8_t* latch) {
  Nvtx nvtx_("vx_read_state_owned");
  if (!h) return fail(VX_ERR_INVALID_ARG, "NULL handle");
  VX_TRY(set_device(h));
  VX_TRY(ensure_owned(h));
  const long long M = (long long)h->owned_ext.size();
  if (M == 0) return VX_OK;
  DevBuf& b = h->stage_ext;
  if (b.bytes < (size_t)M * 13 * 8 + (size_t)M) VX_TRY(b.alloc((size_t)M * 13 * 8 + (size_t)M));
  double* o = b.as<double>();
  uint8_t* ol = reinterpret_cast<uint8_t*>(o + (size_t)M * 13);
  for (const Slab& s : h->slabs) {
    if (!s.own_n) continue;
    if (h->prec == 32)
      k_gather_owned<float><<<grid_of(s.own_n), 256, 0, h->stream>>>(
          make_dev<float>(h, s), s.own_lid.as<long long>(), s.own_gid.as<long long>(), s.own_dst.as<long long>(),
          s.own_n, M, o, ol, h->origin[0], h->origin[1], h->origin[2]);
    else
      k_gather_owned<double><<<grid_of(s.own_n), 256, 0, h->stream>>>(
          make_dev<double>(h, s), s.own_lid.as<long long>(), s.own_gid.as<long long>(), s.own_dst.as<long long>(),
          s.own_n, M, o, ol, h->origin[0], h->origin[1], h->origin[2]);
    VX_CUDA(cudaGetLastError());
  }
  if (pos) VX_CUDA(cudaMemcpyAsync(pos, o, (size_t)M * 24, cudaMemcpyDeviceToHost, h->stream));
  if (quat) VX_CUDA(cudaMemcpyAsync(quat, o + (size_t)M * 3, (size_t)M * 32, cudaMemcpyDeviceToHost, h->stream));
  if (lin) VX_CUDA(cudaMemcpyAsync(lin, o + (size_t)M * 7, (size_t)M * 24, cudaMemcpyDeviceToHost, h->stream));
  if (ang) VX_CUDA(cudaMemcpyAsync(ang, o + (size_t)M * 10, (size_t)M * 24, cudaMemcpyDeviceToHost, h->stream));
  if (latch) VX_CUDA(cudaMemcpyAsync(latch, ol, (size_t)M, cudaMemcpyDeviceToHost, h->stream));
  VX_CUDA(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

vx_status vx_read_voxels(vx_lattice* h, const int64_t* ids, int64_t n, double* pos, double* quat,
                         double* lin, double* ang, uint8_t* latch) {
  Nvtx nvtx_("vx_read_voxels");
  if (!h || (n > 0 && !ids) || n < 0) return fail(VX_ERR_INVALID_ARG, "bad argument");
  if (n == 0) return VX_OK;
  VX_TRY(set_device(h));
  // group the requests by slab
  std::vector<std::vector<int64_t>> which(h->slabs.size());
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= h->N) return fail(VX_ERR_OUT_OF_RANGE, "voxel id out of range");
    const long long x = h->box_of_ext[ids[i]] / h->plane;
    int q = -1;
    for (size_t k = 0; k < h->slabs.size(); ++k)
      if (x >= h->slabs[k].x0 && x < h->slabs[k].x1) q = (int)k;
    if (q < 0) return fail(VX_ERR_OUT_OF_RANGE, "voxel not owned by this rank");
    which[q].push_back(i);
  }
  std::vector<double> hp((size_t)n * 13);
  std::vector<uint8_t> hl((size_t)n);
  for (size_t q = 0; q < h->slabs.size(); ++q) {
    const std::vector<int64_t>& w = which[q];
    const long long m = (long long)w.size();
    if (!m) continue;
    const Slab& s = h->slabs[q];
    std::vector<long long> lid(m), gid(m);
    for (long long i = 0; i < m; ++i) {
      gid[i] = h->box_of_ext[ids[w[i]]];
      lid[i] = gid[i] - s.box_base;
    }
    DevBuf ib, ob;
    VX_TRY(ib.alloc((size_t)m * 16));
    VX_TRY(ob.alloc((size_t)m * 13 * 8 + (size_t)m));
    long long* dl = ib.as<long long>();
    VX_CUDA(cudaMemcpy(dl, lid.data(), (size_t)m * 8, cudaMemcpyHostToDevice));
    VX_CUDA(cudaMemcpy(dl + m, gid.data(), (size_t)m * 8, cudaMemcpyHostToDevice));
    double* o = ob.as<double>();
    uint8_t* ol = reinterpret_cast<uint8_t*>(o + (size_t)m * 13);
    if (h->prec == 32)
      k_read_ids<float><<<grid_of(m), 256, 0, h->stream>>>(make_dev<float>(h, s), dl, dl + m, m, o, o + m * 3, o + m * 7,
                                                           o + m * 10, ol, h->origin[0], h->origin[1], h->origin[2]);
    else
      k_read_ids<double><<<grid_of(m), 256, 0, h->stream>>>(make_dev<double>(h, s), dl, dl + m, m, o, o + m * 3, o + m * 7,
                                                            o + m * 10, ol, h->origin[0], h->origin[1], h->origin[2]);
    VX_CUDA(cudaGetLastError());
    std::vector<double> tmp((size_t)m * 13);
    std::vector<uint8_t> tl((size_t)m);
    VX_CUDA(cudaMemcpyAsync(tmp.data(), o, (size_t)m * 13 * 8, cudaMemcpyDeviceToHost, h->stream));
    VX_CUDA(cudaMemcpyAsync(tl.data(), ol, (size_t)m, cudaMemcpyDeviceToHost, h->stream));
    VX_CUDA(cudaStreamSynchronize(h->stream));
    for (long long i = 0; i < m; ++i) {
      const int64_t t = w[i];
      for (int c = 0; c < 3; ++c) hp[(size_t)t * 3 + c] = tmp[(size_t)i * 3 + c];
      for (int c = 0; c < 4; ++c) hp[(size_t)n * 3 + (size_t)t * 4 + c] = tmp[(size_t)m * 3 + (size_t)i * 4 + c];
      for (int c = 0; c < 3; ++c) hp[(size_t)n * 7 + (size_t)t * 3 + c] = tmp[(size_t)m * 7 + (size_t)i * 3 + c];
      for (int c = 0; c < 3; ++c) hp[(size_t)n * 10 + (size_t)t * 3 + c] = tmp[(size_t)m * 10 + (size_t)i * 3 + c];
      hl[t] = tl[i];
    }
  }
  if (pos) std::memcpy(pos, hp.data(), (size_t)n * 24);
  if (quat) std::memcpy(quat, hp.data() + (size_t)n * 3, (size_t)n * 32);
  if (lin) std::memcpy(lin, hp.data() + (size_t)n * 7, (size_t)n * 24);
  if (ang) std::memcpy(ang, hp.data() + (size_t)n * 10, (size_t)n * 24);
  if (latch) std::memcpy(latch, hl.data(), (size_t)n);
  return VX_OK;
}

double vx_dt(const vx_lattice* h) { return h ? h->dt : 0.0; }
int64_t vx_num_voxels(const vx_lattice* h) { return h ? h->N : -1; }
int64_t vx_num_bonds(const vx_lattice* h) { return h ? h->nbonds : -1; }
int64_t vx_num_surface(const vx_lattice* h) { return h ? h->nsurf : -1; }
int64_t vx_steps_done(const vx_lattice* h) { return h ? h->steps_done : -1; }

int64_t vx_num_contact_pairs(const vx_lattice* h) {
  if (!h || !h->clk.p) return -1;
  if (cudaSetDevice(h->device) != cudaSuccess) return -1;
  Clock c;
  if (cudaMemcpy(&c, h->clk.p, sizeof c, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  long long half = c.npairs;   // half-edges of the rows this handle built
  if (h->nccl()) {             // collective: every rank's rows
    DevBuf t;
    if (t.alloc(8) != VX_OK) return -1;
    if (cudaMemcpy(t.p, &half, 8, cudaMemcpyHostToDevice) != cudaSuccess ||
        ncclAllReduce(t.p, t.p, 1, ncclInt64, ncclSum, h->comm, h->stream) != ncclSuccess ||
        cudaMemcpyAsync(&half, t.p, 8, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
        cudaStreamSynchronize(h->stream) != cudaSuccess)
      return -1;
  }
  return half / 2;
}
int64_t vx_num_rebuilds(const vx_lattice* h) {
  if (!h || !h->clk.p) return -1;
  Clock c;
  if (cudaMemcpy(&c, h->clk.p, sizeof c, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return c.rebuilds;
}
int32_t vx_owned_planes(const vx_lattice* h, int32_t* xb, int32_t* xe) {
  if (!h) return -1;
  if (xb) *xb = h->x0;
  if (xe) *xe = h->x1;
  return h->x1 - h->x0;
}
void* vx_stream(const vx_lattice* h) { return h ? (void*)h->stream : nullptr; }

int64_t vx_contact_pairs(vx_lattice* h, int64_t* pairs, int64_t cap) {
  if (!h) return -1;
  if (!h->collide() || h->tables_dirty || !h->rowptr.p) return 0;
  if (cudaSetDevice(h->device) != cudaSuccess) return -1;
  const int S = (int)h->surf_g.size();
  std::vector<int> rp(S + 1);
  if (cudaMemcpy(rp.data(), h->rowptr.p, (size_t)(S + 1) * 4, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  const long long tot = std::min<long long>(rp[S], h->cap);
  std::vector<int> col((size_t)std::max<long long>(tot, 1));
  if (tot && cudaMemcpy(col.data(), h->col.p, (size_t)tot * 4, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  // external id of every surface index
  std::vector<long long> ext(S, -1);
  for (long long e = 0; e < h->N; ++e) {
    const unsigned g = (unsigned)h->box_of_ext[e];
    auto it = std::lower_bound(h->surf_g.begin(), h->surf_g.end(), g);
    if (it != h->surf_g.end() && *it == g) ext[it - h->surf_g.begin()] = e;
  }
  std::vector<std::pair<long long, long long>> out;
  for (int s = h->rows_begin(); s < h->rows_end(); ++s)
    for (int q = rp[s]; q < std::min<long long>(rp[s + 1], tot); ++q) {
      const long long a = ext[s], b = ext[col[q]];
      out.emplace_back(std::min(a, b), std::max(a, b));
    }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  for (long long i = 0; i < (long long)out.size() && i < cap; ++i) {
    pairs[2 * i] = out[i].first;
    pairs[2 * i + 1] = out[i].second;
  }
  return (int64_t)out.size();
}

vx_status vx_set_instrumentation(vx_lattice* h, int32_t on) {
  if (!h) return fail(VX_ERR_INVALID_ARG, "NULL handle");
  h->instr = on != 0;
  h->instr_stride = on > 1 ? on : 1;
  for (int i = 0; i < 4; ++i) { h->t_ms[i] = 0; h->t_cnt[i] = 0; }
  return VX_OK;
}
vx_status vx_kernel_times(vx_lattice* h, double out_ms[4], int64_t counts[4]) {
  if (!h) return fail(VX_ERR_INVALID_ARG, "NULL handle");
  for (int i = 0; i < 4; ++i) {
    if (out_ms) out_ms[i] = h->t_ms[i];
    if (counts) counts[i] = h->t_cnt[i];
  }
  return VX_OK;
}
int32_t vx_launches_per_step(const vx_lattice* h) { return h ? h->launches_per_step() : -1; }

vx_status vx_set_batch(vx_lattice* h, int32_t stride) {
  if (!h || stride < 0) return fail(VX_ERR_INVALID_ARG, "bad argument");
  if (stride > 0) {
    if (stride < 2) return fail(VX_ERR_INVALID_ARG, "a batched scene needs >= 1 plane + a separator");
    // every stride-th plane (stride-1, 2 stride-1, ...) must be empty
    for (int x = stride - 1; x < h->nx; x += stride)
      for (long long c = 0; c < (long long)h->ny * h->nz; ++c) {
        const long long j = c % h->ny, k = c / h->ny;
        if (h->cells[(size_t)x + (size_t)h->nx * ((size_t)j + (size_t)h->ny * k)])
          return fail(VX_ERR_INVALID_ARG, "separator plane x=" + std::to_string(x) + " is not empty");
      }
  }
  h->batch_stride = stride;
  h->clear_graphs();
  VX_TRY(set_device(h));
  return set_force_rebuild(h);
}
vx_status vx_set_batch_z(vx_lattice* h, int32_t stride) {
  if (!h || stride < 0) return fail(VX_ERR_INVALID_ARG, "bad argument");
  if (stride > 0) {
    if (stride < 2) return fail(VX_ERR_INVALID_ARG, "a z-stacked scene needs >= 1 layer + a separator");
    // every stride-th layer (stride-1, 2 stride-1, ...) must be empty
    const size_t layer = (size_t)h->nx * h->ny;
    for (int z = stride - 1; z < h->nz; z += stride)
      for (size_t c = 0; c < layer; ++c)
        if (h->cells[c + layer * (size_t)z])
          return fail(VX_ERR_INVALID_ARG, "separator layer z=" + std::to_string(z) + " is not empty");
  }
  h->batch_stride_z = stride;
  h->clear_graphs();
  VX_TRY(set_device(h));
  return set_force_rebuild(h);
}
vx_status vx_set_batch_y(vx_lattice* h, int32_t stride) {
  if (!h || stride < 0) return fail(VX_ERR_INVALID_ARG, "bad argument");
  if (stride > 0) {
    if (stride < 2) return fail(VX_ERR_INVALID_ARG, "a y-stacked scene needs >= 1 row + a separator");
    // every stride-th row (stride-1, 2 stride-1, ...) must be empty
    for (int y = stride - 1; y < h->ny; y += stride)
      for (int z = 0; z < h->nz; ++z)
        for (int x = 0; x < h->nx; ++x)
          if (h->cells[(size_t)x + (size_t)h->nx * ((size_t)y + (size_t)h->ny * z)])
            return fail(VX_ERR_INVALID_ARG, "separator row y=" + std::to_string(y) + " is not empty");
  }
  h->batch_stride_y = stride;
  h->clear_graphs();
  VX_TRY(set_device(h));
  return set_force_rebuild(h);
}
int32_t vx_num_scenes(const vx_lattice* h) {
  if (!h) return -1;
  const int kx = h->batch_stride ? (h->nx + h->batch_stride - 1) / h->batch_stride : 1;
  const int ky = h->batch_stride_y ? (h->ny + h->batch_stride_y - 1) / h->batch_stride_y : 1;
  const int kz = h->batch_stride_z ? (h->nz + h->batch_stride_z - 1) / h->batch_stride_z : 1;
  return kx * ky * kz;
}

vx_status vx_set_engine(vx_lattice* h, int32_t engine) {
  if (!h) return fail(VX_ERR_INVALID_ARG, "NULL handle");
  if (engine != VX_ENGINE_TWO_PASS && engine != VX_ENGINE_FUSED && engine != VX_ENGINE_AUTO)
    return fail(VX_ERR_INVALID_ARG, "unknown engine");
  h->engine_req = engine;
  h->engine_resolved = false;
  if (engine != VX_ENGINE_AUTO) h->engine = engine;
  h->clear_graphs();
  return VX_OK;
}
int32_t vx_get_engine(const vx_lattice* h) {
  if (!h) return -1;
  return h->engine_req == VX_ENGINE_AUTO && !h->engine_resolved ? VX_ENGINE_AUTO : h->engine;
}

}  // extern "C"
