/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU reference ("oracle") for the per-timestep method of
 * Hiller & Lipson, "Dynamic Simulation of Soft Heterogeneous Objects"
 * (arXiv:1212.2845).  Citations "P:n" are line numbers of the paper text
 * (/root/reference/PAPER.md at survey time); readings of ambiguous passages
 * follow SURVEY.md §8(c) and are listed in DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no source, header,
 * table or helper with the CUDA product path (paper_1212_2845_b200/).
 *
 * Voxel ids are the filled cells of the input grid in x-fastest order.
 */
#ifndef VOXEL_ORACLE_H
#define VOXEL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_sim orc_sim;

typedef struct {
  double E;      /* elastic modulus, Pa            (App. B AddMat) */
  double nu;     /* Poisson ratio                    */
  double rho;    /* density, kg/m^3                                           */
  double cte;    /* thermal expansion coefficient                */
  double mu_s;   /* static friction coefficient                    */
  double mu_d;   /* dynamic friction coefficient                    */
} orc_material;

typedef struct {
  double gravity;        /* m/s^2, acts along -z                    */
  int32_t floor_on;      /* 1: floor plane z = floor_z present      */
  double floor_z;
  double T_ref, T_amp, T_freq, T_phase; /* T_n = T_ref + T_amp sin(2 pi f t_n + phase) */
  double zeta_bond;      /* Eq. 34-35 (SetBondDampZ)                 */
  double zeta_ground;    /* SetSlowDampZ                            */
  double zeta_col;       /* SetCollisionDampZ                       */
  double horizon_voxels; /* not used by the oracle (all-pairs every step)   */
  double dt_safety;      /* multiplies the Eq. 31 bound                     */
  int32_t self_collision;/* 1: surface-voxel self collision     */
} orc_env;

/* Create a simulation from a dense grid (x-fastest, 0 = empty, k -> mats[k-1]).
 * Returns NULL on invalid input (message via orc_last_error()). */
orc_sim* orc_create(int32_t nx, int32_t ny, int32_t nz, double l, const double origin[3],
                    const uint8_t* cells, const orc_material* mats, int32_t nmat,
                    const orc_env* env);
void orc_destroy(orc_sim* s);
const char* orc_last_error(void);

int64_t orc_num_voxels(const orc_sim* s);
int64_t orc_num_bonds(const orc_sim* s);
int64_t orc_num_surface(const orc_sim* s);
double orc_dt(const orc_sim* s);

/* fixed: N bytes or NULL; fext: 3N doubles or NULL (replaces previous). */
int orc_set_boundary(orc_sim* s, const uint8_t* fixed, const double* fext);
/* App. B AddFixedRegion / AddForcedRegion; kind 0 = fixed, 1 = forced. */
int orc_add_region(orc_sim* s, int32_t kind, const double origin[3], const double size[3],
                   const double force[3]);
int orc_set_state(orc_sim* s, const double* pos, const double* quat, const double* linmom,
                  const double* angmom, const uint8_t* latch);
int orc_read_state(const orc_sim* s, double* pos, double* quat, double* linmom,
                   double* angmom, uint8_t* latch);
int orc_set_step(orc_sim* s, int64_t n);
int64_t orc_get_step(const orc_sim* s);
int orc_set_threads(orc_sim* s, int32_t n);
/* Override the stable step (used when a sub-lattice stands in for a
 * neighbourhood of a larger lattice whose Eq. 31 dt differs). */
int orc_set_dt(orc_sim* s, double dt);
/* Advance n steps.  0 ok, -6 diverged (message names voxel and step). */
int orc_step(orc_sim* s, int64_t n);

/* ---- granular entry points used by the pin tests ------------------------ */
/* Eq. 1-3: out = {E_c, G_c, mu_c}. */
void orc_composite(double E1, double nu1, double E2, double nu2, double out[3]);
/* Eq. 4-12: out = {a1, a2, b1, b2, b3}. */
void orc_beam_constants(double Ec, double Gc, double l, double out[5]);
/* Loads of one bond (axis 0/1/2, a on the negative side) in world frame:
 * out = {Fa[3], Ma[3], Fb[3], Mb[3]}.  State layout per voxel:
 * D[3], q[4] (w,x,y,z), P[3], phi[3]. */
void orc_bond_loads(const orc_sim* s, int32_t a_mat, int32_t b_mat, int32_t axis,
                    const double* state_a, const double* state_b, double dT, double out[12]);
/* Overlapping contact pairs (a<b) at the current state (all-pairs definition).
 * Writes up to cap pairs, returns the total count. */
int64_t orc_contact_pairs(const orc_sim* s, int32_t* pairs, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
