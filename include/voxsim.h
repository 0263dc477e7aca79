/*
 * voxsim.h -- C ABI of the B200-native voxel soft-body stepper
 * (Hiller & Lipson, "Dynamic Simulation of Soft Heterogeneous Objects",
 * arXiv:1212.2845).  "P:n" cites line n of the paper text;
 * "§8(c) Rn" cites the reading n listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Plain C types only.  Every host pointer is owned by the caller and is
 *    copied during the call; the library never retains it.  Device memory is
 *    owned by the library and released by vx_destroy().
 *  - Voxel order at the boundary ("external ids") = the filled cells of the
 *    input grid in x-fastest order (x fastest, then y, then z).
 *  - Units SI; orientations are unit quaternions (w, x, y, z).
 *  - Every call returns a vx_status (or a plain value for the queries); a
 *    failing call leaves a message in vx_last_error() (thread-local) and
 *    leaves the lattice unchanged unless stated otherwise.  No C++ exception
 *    crosses the ABI.
 *  - There is no CPU fallback: without a CUDA device vx_create_lattice
 *    returns VX_ERR_NO_DEVICE.
 *  - Calls on one handle must be serialised by the caller.  With nranks > 1
 *    every rank makes the same sequence of calls (collective semantics).
 */
#ifndef VOXSIM_H
#define VOXSIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VOXSIM_ABI_VERSION 3   /* 2: vx_prepare_steps, vx_set_batch_y/_z, VX_ENGINE_AUTO default;
                                  3: owned-voxel state I/O (vx_num_owned ...) */

typedef struct vx_lattice vx_lattice; /* opaque, library-owned */

typedef enum {
  VX_OK = 0,
  VX_ERR_INVALID_ARG = -1,  /* bad argument or violated material / env invariant */
  VX_ERR_OUT_OF_RANGE = -2, /* cell or material index out of range (App. B SetMat) */
  VX_ERR_CUDA = -3,         /* CUDA runtime error (message has the CUDA string) */
  VX_ERR_NCCL = -4,         /* NCCL error (nranks > 1) */
  VX_ERR_OOM = -5,          /* device allocation failed */
  VX_ERR_DIVERGED = -6,     /* non-finite state; message names voxel id and step */
  VX_ERR_STATE = -7,        /* call out of order (e.g. step before set_materials) or an
                               internal capacity (contact pair list) exceeded */
  VX_ERR_NO_DEVICE = -8     /* no CUDA device visible */
} vx_status;

/* Lattice geometry (App. B CVX_Object::InitializeMatter / SetMat). */
typedef struct {
  int32_t nx, ny, nz;       /* workspace size in voxels (>= 1 each)                   */
  double lattice_dim;       /* l, m, > 0 (beam length = voxel pitch)            */
  double origin[3];         /* position of the corner of cell (0,0,0); voxel (i,j,k)'s
                               rest centre is origin + l (i+1/2, j+1/2, k+1/2)          */
  const uint8_t* cells;     /* nx*ny*nz, x-fastest; 0 = empty, k>=1 -> palette[k-1]    */
  int32_t precision;        /* 32 or 64: arithmetic type of the device path            */
  int32_t device;           /* CUDA device ordinal                                     */
  int32_t rank, nranks;     /* slab decomposition along x (nranks >= 1, <= nx)         */
  const void* nccl_id;      /* 128-byte ncclUniqueId from vx_nccl_unique_id() on rank 0,
                               broadcast by the caller: one process per GPU, ghost planes
                               by NCCL send/recv.  One id serves one lattice (as with
                               ncclCommInitRank): create a new id for every lattice.  NULL with nranks > 1 (rank 0): the
                               nranks slabs are emulated inside this one handle on one
                               device (ghost planes by device copies) -- the same slab
                               arithmetic, used to test bitwise slab invariance.        */
} vx_lattice_desc;

/* Planes [x_begin, x_end) of the x-slab of `rank` out of `nranks` over nx
 * planes (balanced: floor(r nx / P) .. floor((r+1) nx / P)).  Host-only. */
vx_status vx_slab_planes(int32_t nx, int32_t nranks, int32_t rank, int32_t* x_begin,
                         int32_t* x_end);

/* Material palette entry (App. B AddMat).
 * Invariants: E > 0, rho > 0, -1 < nu < 0.5, mu_s >= mu_d >= 0. */
typedef struct {
  double E;     /* elastic modulus, Pa                         */
  double nu;    /* Poisson ratio (G = E / (2(1+nu)))    */
  double rho;   /* density, kg/m^3 (m = rho l^3, I = m l^2/6)  */
  double cte;   /* coefficient of thermal expansion, 1/K (Eq. 40) */
  double mu_s;  /* static friction coefficient (Eq. 36) */
  double mu_d;  /* dynamic friction coefficient (Eq. 37-38)    */
} vx_material;

/* Environment and solver settings (App. B CVX_Environment / CVX_Sim setters,
 * P:545-618).  Damping ratios must lie in [0,1]. */
typedef struct {
  double gravity;        /* m/s^2 along -z                                  */
  int32_t floor_on;      /* floor plane z = floor_z                          */
  double floor_z;
  double T_ref;          /* temperature schedule T_n = T_ref + T_amp sin(2 pi T_freq t_n
                            + T_phase), t_n = n dt                        */
  double T_amp, T_freq, T_phase;
  double zeta_bond;      /* bond damping ratio (Eq. 34-35, SetBondDampZ)             */
  double zeta_ground;    /* ground damping ratio (SetSlowDampZ)               */
  double zeta_col;       /* collision damping ratio (SetCollisionDampZ)       */
  double horizon_voxels; /* collision horizon in voxels (2)                   */
  double dt_safety;      /* multiplies the stable step of Eq. 31; in (0,1]           */
  int32_t self_collision;/* surface-voxel self collision                 */
} vx_env;

/* Create a lattice on desc->device (collective over nranks if nranks > 1).
 * Builds the voxel ids, bond slots, surface list and neighbour masks (P:100,
 * P:189).  Initial state: every voxel at rest on its lattice site with
 * identity orientation.  Errors: INVALID_ARG, OUT_OF_RANGE (cell > 255 never
 * happens; material indices are validated in vx_set_materials), NO_DEVICE,
 * CUDA, NCCL, OOM.  On error *out is NULL. */
vx_status vx_create_lattice(const vx_lattice_desc* desc, vx_lattice** out);

/* Palette of n materials (n >= max cell index).  Validates the invariants,
 * builds the material and material-pair tables (Eq. 1-12, composite E_c,
 * G_c; beam constants a1..b3; damping coefficients), and selects the stable
 * timestep with a device max-reduction (Eq. 31-32; §8(c) R9).
 * Errors: INVALID_ARG (invariant violated), OUT_OF_RANGE (a cell references
 * a material index > n). */
vx_status vx_set_materials(vx_lattice* h, const vx_material* palette, int32_t n);

/* Environment and solver settings.  Errors: INVALID_ARG (damping ratio
 * outside [0,1], dt_safety outside (0,1], horizon <= 0).  Self collision
 * works with any slab count: each step every slab's surface-voxel state
 * (32 B fp32 / 64 B fp64 per surface voxel) is broadcast to every rank, the
 * motion budget takes the max |V| over all ranks (one allreduce), and each
 * rank builds the shortlist rows of its own surface voxels;
 * results are bitwise independent of the slab count. */
vx_status vx_set_environment(vx_lattice* h, const vx_env* env);

/* Per-voxel boundary conditions in external order, replacing previous ones:
 * fixed[N] (nonzero = kinematic, never integrated, loads dropped) or
 * NULL for none; f_ext[3N] external force in N or NULL for none. */
vx_status vx_set_boundary(vx_lattice* h, const uint8_t* fixed, const double* f_ext);

/* App. B AddFixedRegion / AddForcedRegion: origin and size are
 * fractions [0,1] of the workspace; a voxel belongs to the region if its cell
 * box overlaps the region box with positive measure (or, for a zero-width
 * region axis, the plane lies within the closed cell interval).  kind 0 =
 * fixed, 1 = forced: `force` (N) is divided equally among every filled voxel
 * touched and added to their external force.  Fixed takes precedence.
 * Errors: INVALID_ARG (kind, or origin/size outside [0,1]). */
vx_status vx_add_region(vx_lattice* h, int32_t kind, const double origin[3],
                        const double size[3], const double force[3]);

/* Replace the dynamic state (external order; any pointer may be NULL to keep
 * that part): pos[3N] absolute positions D (m), quat[4N] (w,x,y,z) unit
 * quaternions, linmom[3N] P (kg m/s), angmom[3N] phi (kg m^2/s), latch[N]
 * static-friction flags.  Resets the collision pair list. */
vx_status vx_set_state(vx_lattice* h, const double* pos, const double* quat,
                       const double* linmom, const double* angmom, const uint8_t* latch);

/* Exact checkpoint of this rank's device state (displacements, orientations,
 * momenta, latch bits, step counter, motion budget), for bitwise resume:
 * load(save(x)) then step(k) equals the uninterrupted run bit for bit.
 * (vx_read_state / vx_set_state go through absolute fp64 positions and are
 * exact only to rounding.)  The buffer is caller-owned host memory of
 * vx_checkpoint_bytes() bytes; load checks the lattice shape and precision
 * (INVALID_ARG on mismatch). */
int64_t vx_checkpoint_bytes(const vx_lattice* h);
vx_status vx_save_checkpoint(vx_lattice* h, void* buf, int64_t bytes);
vx_status vx_load_checkpoint(vx_lattice* h, const void* buf, int64_t bytes);

/* Set the step counter n (time t_n = n dt of the temperature schedule). */
vx_status vx_set_step(vx_lattice* h, int64_t n);

/* Build, without running them, the CUDA graphs vx_step(h, n) will replay from
 * the current state (and resolve VX_ENGINE_AUTO, tune the launch geometry,
 * pack the surface table): the state does not advance.  Optional -- vx_step
 * does the same on first use; calling this first keeps graph construction out
 * of a timed region.  Graphs depend on n modulo 32 steps, the state-copy parity
 * and the instrumentation setting, so call it after vx_set_instrumentation.
 * Errors: INVALID_ARG for n < 0; STATE before materials/environment are set. */
vx_status vx_prepare_steps(vx_lattice* h, int64_t n);

/* Advance n steps (n >= 0) of the synchronous two-phase update:
 * bond loads from the frozen state (Eq. 13-24, 33-35, 39-40), per-voxel
 * fixed-order sums (Eq. 25-26), gravity, ground damping, self collision,
 * floor and friction, integration (Eq. 27-30).  Blocks until the
 * n steps are done.  Errors: STATE (before set_materials), DIVERGED (the state
 * is left as computed; the message names the first diverged external voxel
 * id and the step), CUDA, NCCL. */
vx_status vx_step(vx_lattice* h, int64_t n);

/* Copy the full state to host arrays (external order; NULL skips a part):
 * pos[3N], quat[4N], linmom[3N], angmom[3N], latch[N].  With nranks > 1 each
 * rank receives the global state (collective). */
vx_status vx_read_state(vx_lattice* h, double* pos, double* quat, double* linmom,
                        double* angmom, uint8_t* latch);

/* Copy the state of n selected voxels (external ids[n]) to host arrays of n
 * entries each (layout as vx_read_state).  Errors: OUT_OF_RANGE (an id not in
 * [0,N) or not owned by this rank when nranks > 1). */
vx_status vx_read_voxels(vx_lattice* h, const int64_t* ids, int64_t n, double* pos,
                         double* quat, double* linmom, double* angmom, uint8_t* latch);

/* Owned-voxel state I/O (one rank per GPU, nranks > 1): the voxels of this
 * handle's x-slab (vx_owned_planes), in ascending external id -- each rank
 * moves only its own share of the state instead of the global arrays.  No
 * collective; with nranks = 1 (or emulated slabs) the owned voxels are all N.
 * The state lives in the slab's owned planes; ghost planes are refreshed from
 * the neighbours by every step's exchange, so setting the owned
 * voxels on every rank sets the global state.
 *   vx_num_owned: M (>= 0; -1 on a NULL handle)
 *   vx_owned_ids: the M external ids into ids[M] (caller-owned)
 *   vx_set_state_owned / vx_read_state_owned: arrays of M entries in that
 *     order, layout as vx_set_state / vx_read_state (NULL skips a part; a
 *     set also forces a collision rebuild).  Errors: INVALID_ARG (NULL handle),
 *     CUDA. */
int64_t vx_num_owned(const vx_lattice* h);
vx_status vx_owned_ids(const vx_lattice* h, int64_t* ids);
vx_status vx_set_state_owned(vx_lattice* h, const double* pos, const double* quat,
                             const double* linmom, const double* angmom, const uint8_t* latch);
vx_status vx_read_state_owned(vx_lattice* h, double* pos, double* quat, double* linmom,
                              double* angmom, uint8_t* latch);

/* Queries (plain values; 0 / -1 on a NULL handle). */
double vx_dt(const vx_lattice* h);                 /* stable timestep (s), 0 before set_materials */
int64_t vx_num_voxels(const vx_lattice* h);        /* N, global                     */
int64_t vx_num_bonds(const vx_lattice* h);         /* face-adjacent pairs, global   */
int64_t vx_num_surface(const vx_lattice* h);       /* surface voxels, global */
int64_t vx_steps_done(const vx_lattice* h);        /* step counter n                 */
int64_t vx_num_contact_pairs(const vx_lattice* h); /* current shortlist size (pairs a<b);
                                                      collective over NCCL ranks */
int64_t vx_num_rebuilds(const vx_lattice* h);      /* broadphase rebuilds so far     */
int32_t vx_owned_planes(const vx_lattice* h, int32_t* x_begin, int32_t* x_end); /* this rank's x-slab */

/* Copy the current collision shortlist as external-id pairs (a < b),
 * ascending, into pairs[2*cap]; returns the total number of pairs (which may
 * exceed cap), 0 when self collision is off, -1 on error.  The list holds
 * every surface pair within the horizon cutoff at the last rebuild; over NCCL
 * ranks, the pairs with at least one voxel in this rank's slab. */
int64_t vx_contact_pairs(vx_lattice* h, int64_t* pairs, int64_t cap);

/* The CUDA stream every kernel of this lattice is launched on (cudaStream_t).
 * Owned by the library; valid until vx_destroy. */
void* vx_stream(const vx_lattice* h);

/* Kernel-level instrumentation.  on = 0: off; on = 1: the CUDA graphs vx_step
 * replays carry CUDA event-record nodes around every launch class of every
 * step (on vx_stream()); on = n > 1: of every n-th step.  The times of one
 * graph replay are read while the next one runs; vx_kernel_times returns,
 * since the last reset, the summed device time in ms and the launch count of
 * each kernel class: out_ms[0]/counts[0] = K3 bonds, [1] = K4
 * gather-integrate or the fused pass, [2] = other (clock, surface table,
 * broadphase, contact, ghost-plane copies), [3] = the whole step. */
vx_status vx_set_instrumentation(vx_lattice* h, int32_t on);
vx_status vx_kernel_times(vx_lattice* h, double out_ms[4], int64_t counts[4]);
/* Number of kernels vx_step launches per step with the current settings. */
int32_t vx_launches_per_step(const vx_lattice* h);

/* Step engine.  VX_ENGINE_TWO_PASS: the bond kernel K3 writes per-bond load
 * records to HBM and the gather-integrate kernel K4 reads them ("forces
 * … calculated separately, then … summed"; 384 B/voxel-step in fp32).
 * VX_ENGINE_FUSED: one kernel per step sweeps x-planes, keeps every bond's
 * loads on chip and writes S_{n+1} to a second state copy (112 B/voxel-step);
 * same arithmetic per bond and per voxel, same summation order.  Any nz
 * (taller than 256: z chunks of 256 voxels, each recomputing the -z bond of
 * its lowest layer).  In kernel timing (vx_kernel_times) the fused kernel is
 * reported in slot [1].
 * VX_ENGINE_AUTO (the default): resolved once, at the first vx_step, to the
 * faster of the two for this lattice -- fused when nz >= 64 and the lattice
 * has >= 2^22 cells, or when it is split into slabs (then fused unless a
 * plane has fewer than 32 cells, the same choice on every rank);
 * otherwise both are timed on the current state (as CUDA graphs, without
 * advancing it) and the faster kept.  vx_get_engine returns VX_ENGINE_AUTO
 * until it is resolved, then the engine in use.  Errors: INVALID_ARG for any
 * other value. */
typedef enum { VX_ENGINE_TWO_PASS = 0, VX_ENGINE_FUSED = 1, VX_ENGINE_AUTO = 2 } vx_engine;

/* Batched independent scenes (the design-automation use of
 * "many, many physical evaluations"): the caller packs K scenes along x,
 * scene s in planes [s*stride, s*stride + stride - 1) and an empty separator
 * plane after each (no bonds cross it).  Declaring the stride makes self
 * collision ignore pairs of different scenes, so every scene evolves exactly
 * as it would alone (up to its x offset) while one launch steps all of them.
 * stride 0 = one scene.  Errors: INVALID_ARG if a separator plane is not
 * empty.  All scenes share the environment, the time step and the clock. */
vx_status vx_set_batch(vx_lattice* h, int32_t stride);
/* Scenes stacked along z as well: every `stride` layers one scene, layer
 * stride-1 of each block empty (no bonds cross it).  The fused engine runs one
 * thread per z, so shallow scenes (nz < 32) stacked up to ~256 layers keep its
 * warps full.  The floor of each stacked scene lies under its own
 * lowest layer: its penetration is measured from the layer index within the
 * block (k mod stride), so each scene sees what it would alone; self collision
 * ignores pairs of different z blocks.  stride 0 = no z stacking.  Errors:
 * INVALID_ARG if a separator layer is not empty.  vx_num_scenes counts x
 * blocks times y blocks times z blocks. */
vx_status vx_set_batch_z(vx_lattice* h, int32_t stride);
/* Scenes stacked along y as well: every `stride` rows one scene, row stride-1
 * of each block empty.  The physics is invariant under a y translation; self
 * collision ignores pairs of different y blocks.  For scenes whose y-z plane
 * is smaller than a warp (ny * nz < 32, e.g. a 10 x 1 x 1 cantilever) y
 * stacking gives the (y, z)-mapped fused pass full warps.  stride 0 = none.
 * Errors: INVALID_ARG if a separator row is not empty. */
vx_status vx_set_batch_y(vx_lattice* h, int32_t stride);
int32_t vx_num_scenes(const vx_lattice* h);
vx_status vx_set_engine(vx_lattice* h, int32_t engine);
int32_t vx_get_engine(const vx_lattice* h);

/* Release all device memory and the communicator. NULL is a no-op. */
void vx_destroy(vx_lattice* h);

/* Thread-local message of the last failing call ("" if none). */
const char* vx_last_error(void);

/* Fill 128 bytes with a fresh ncclUniqueId (call on rank 0 only). */
vx_status vx_nccl_unique_id(void* out128);

/* ABI version (VOXSIM_ABI_VERSION). */
int32_t vx_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VOXSIM_H */
