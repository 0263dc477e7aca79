"""Closed-form pins of the oracle's damping, rotation and thermal terms.

Each test reduces the oracle to a system whose exact discrete trajectory is
known in closed form from the paper's integration rule (Eq. 27-30)
and the term under test, and checks the oracle against it.  A one-symbol slip
in the term (a factor 2 in c_t or c_r, m_max for m_min, SPEC's k_phi = 2 b3
for a2, I != m l^2 / 6, the product order of Eq. 30's rotation update, the
thermal mean of Eq. 40 replaced by one voxel's alpha, the harmonic-mean
contact stiffness, ...) fails at least one of them.  CPU only.

    Bond damping   Eq. 33-35, readings R10 (m_min, I_min), R11 (k_phi = a2)
    Ground damping P:254, App. B, reading R12
    Floor          P:258-274, reading R14 (k_f = E l, zeta_col normal damping)
    Contact        reading R16
    Rotation       Eq. 30, readings R6 (quaternion) and R8 (I = m l^2 / 6)
    Thermal        Eq. 39-40, rest length l (1 + (alpha_a + alpha_b)/2 dT)
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import workloads as W
from oracle import OracleSim

L = 1e-3


def mat(E=1e6, nu=0.35, rho=1000.0, cte=0.0, mu_s=0.0, mu_d=0.0):
    return dict(E=E, nu=nu, rho=rho, cte=cte, mu_s=mu_s, mu_d=mu_d)


def sim(cells, mats, **env):
    e = W._env(**env)
    cells = np.asarray(cells, np.uint8)
    s = W.Scene("pin", cells, L, mats, e)
    o = OracleSim(cells, L, mats, e)
    o.set_state(*s.initial_state())
    return o, s


def harmonic(a, b):
    """Eq. 1 / Eq. 2 composite: 2 a b / (a + b)."""
    return 2 * a * b / (a + b)


def _damped_pair_trajectory(k, beta, dt, e0, v0, n):
    """Exact iterates of the damped symplectic-Euler relative coordinate:
    v' = beta v - k e,  e' = e + dt v'  (A = [[1 - dt k, dt beta], [-k, beta]]),
    evaluated as matrix powers; also the eigenvalues of A."""
    A = np.array([[1 - dt * k, dt * beta], [-k, beta]])
    x = np.array([e0, v0])
    out = []
    P = np.eye(2)
    for _ in range(n + 1):
        out.append(P @ x)
        P = A @ P
    return np.array(out), np.linalg.eigvals(A)


# --------------------------------------------------------------- Eq. 33-35
@pytest.mark.parametrize("zeta", [0.3, 1.0])
def test_bond_damping_axial_pair_closed_form(zeta):
    """Two free voxels of different density on an x-bond, pure axial motion.
    The a-frame stays the identity, so X2 = x_b - x_a - l exactly and the
    loads reduce to F_a = a1 X2 + c_t (V_b - V_a)/2 (Eq. 33: V_r = V_b - V_avg,
    no spin).  Relative coordinate e = X2, v = V_b - V_a, with
    mu^-1 = 1/m_a + 1/m_b:  v' = (1 - dt c_t mu^-1 / 2) v - dt a1 mu^-1 e,
    e' = e + dt v'.  c_t = 2 zeta sqrt(m_min a1) (Eq. 34, R10)."""
    Ea, Eb, ra, rb = 1e6, 3e6, 1000.0, 2500.0
    o, s = sim(np.array([[[1, 2]]]), [mat(E=Ea, rho=ra), mat(E=Eb, rho=rb)], zeta_bond=zeta)
    ma, mb = ra * L ** 3, rb * L ** 3
    a1 = harmonic(Ea, Eb) * L * L / L                      # Eq. 8: E_c A / l
    ct = 2 * zeta * math.sqrt(min(ma, mb) * a1)            # Eq. 34, m = m_min
    dt = o.dt
    assert dt == pytest.approx(1 / (2 * math.pi * math.sqrt(a1 / min(ma, mb))), rel=1e-14)
    mu_inv = 1 / ma + 1 / mb
    k = dt * a1 * mu_inv
    beta = 1 - dt * ct * mu_inv / 2
    pos, quat, P, phi, latch = s.initial_state()
    e0, v0 = 3e-6, -2e-3                                   # stretched, closing
    pos[1, 0] += e0
    P[1, 0] = mb * v0                                      # V_a = 0, V_b = v0
    o.set_state(pos, quat, P, phi, latch)
    n = 300
    ref, lam = _damped_pair_trajectory(k, beta, dt, e0, v0, n)
    got = []
    for _ in range(n + 1):
        st = o.read_state()
        got.append([st.pos[1, 0] - st.pos[0, 0] - L, st.linmom[1, 0] / mb - st.linmom[0, 0] / ma])
        o.step(1)
    got = np.array(got)
    assert np.abs(got[:, 0] - ref[:, 0]).max() <= 1e-9 * e0
    assert np.abs(got[:, 1] - ref[:, 1]).max() <= 1e-9 * abs(v0)
    # the per-step decay |lambda|^2 = det A = beta (complex pair) is what damping sets
    assert np.prod(lam).real == pytest.approx(beta, rel=1e-12)
    # total momentum is untouched (equal and opposite loads)
    st = o.read_state()
    assert abs(st.linmom[:, 0].sum() - mb * v0) <= 1e-12 * mb * abs(v0)


@pytest.mark.parametrize("zeta", [0.3, 1.0])
def test_bond_damping_torsion_pair_closed_form(zeta):
    """Two free voxels twisted about their common x-bond.  Rotations about one
    axis commute, the a-frame keeps the bond on x (X2 = Y2 = Z2 = 0), the
    relative rotation is psi = psi_b - psi_a about x and only the torsional
    pair acts: M_a.x = a2 psi + c_r (w_b - w_a)/2, M_b = -M_a.  With
    I = m l^2 / 6 (R8), iota = 1/I_a + 1/I_b, c_r = 2 zeta sqrt(I_min a2)
    (Eq. 35, R10, R11 k_phi = a2 = G_c J / l, J = l^4/6):
    W' = (1 - dt c_r iota / 2) W - dt a2 iota psi,  psi' = psi + dt W'."""
    Ea, Eb, ra, rb, nua, nub = 1e6, 4e6, 1000.0, 1800.0, 0.3, 0.45
    o, s = sim(np.array([[[1, 2]]]), [mat(E=Ea, rho=ra, nu=nua), mat(E=Eb, rho=rb, nu=nub)],
               zeta_bond=zeta)
    ma, mb = ra * L ** 3, rb * L ** 3
    Ia, Ib = ma * L * L / 6, mb * L * L / 6
    Gc = harmonic(Ea / (2 * (1 + nua)), Eb / (2 * (1 + nub)))   # Eq. 2, G = E / (2 (1 + nu))
    a2 = Gc * (L ** 4 / 6) / L                                   # Eq. 9 with Eq. 5
    cr = 2 * zeta * math.sqrt(min(Ia, Ib) * a2)
    dt = o.dt
    iota = 1 / Ia + 1 / Ib
    k = dt * a2 * iota
    beta = 1 - dt * cr * iota / 2
    pos, quat, P, phi, latch = s.initial_state()
    psi0, w0 = 2e-3, 30.0                                  # rad, rad/s (voxel b)
    quat[1] = [math.cos(psi0 / 2), math.sin(psi0 / 2), 0.0, 0.0]
    phi[1, 0] = Ib * w0
    o.set_state(pos, quat, P, phi, latch)
    n = 300
    ref, _ = _damped_pair_trajectory(k, beta, dt, psi0, w0, n)
    got = []
    for _ in range(n + 1):
        st = o.read_state()
        ang = 2 * np.arctan2(st.quat[:, 1], st.quat[:, 0])    # rotation about x
        assert np.abs(st.quat[:, 2:]).max() <= 1e-15
        got.append([ang[1] - ang[0], st.angmom[1, 0] / Ib - st.angmom[0, 0] / Ia])
        assert np.abs(st.pos - pos).max() <= 1e-18            # no force at all
        o.step(1)
    got = np.array(got)
    assert np.abs(got[:, 0] - ref[:, 0]).max() <= 1e-9 * psi0
    assert np.abs(got[:, 1] - ref[:, 1]).max() <= 1e-9 * abs(w0)


def test_bond_damping_is_absent_at_zero_zeta():
    """zeta_b = 0: the same axial pair is the undamped recurrence (beta = 1)."""
    o, s = sim(np.array([[[1, 1]]]), [mat()], zeta_bond=0.0)
    m = 1e-6
    a1 = 1e6 * L
    pos, quat, P, phi, latch = s.initial_state()
    pos[1, 0] += 1e-6
    o.set_state(pos, quat, P, phi, latch)
    ref, lam = _damped_pair_trajectory(o.dt * a1 * 2 / m, 1.0, o.dt, 1e-6, 0.0, 200)
    o.step(200)
    st = o.read_state()
    assert st.pos[1, 0] - st.pos[0, 0] - L == pytest.approx(ref[-1, 0], abs=1e-9 * 1e-6)
    assert np.abs(lam) == pytest.approx([1.0, 1.0], rel=1e-12)


# --------------------------------------------------------------- ground damping
def test_ground_damping_translational_geometric_decay():
    """A free voxel (no bond, no gravity) with zeta_g > 0: F = -c_g V with
    c_g = 2 zeta_g sqrt(m E l) (R12), so P_n = P_0 (1 - dt c_g / m)^n
    and D_n = D_0 + dt / m * sum_{q=1..n} P_q."""
    E, rho, zg = 3e6, 1300.0, 0.2
    o, s = sim(np.ones((1, 1, 1)), [mat(E=E, rho=rho)], zeta_ground=zg)
    m = rho * L ** 3
    dt = o.dt
    assert dt == pytest.approx(1 / (2 * math.pi * math.sqrt(E * L / m)), rel=1e-14)
    cg = 2 * zg * math.sqrt(m * E * L)
    f = 1 - dt * cg / m
    pos, quat, P, phi, latch = s.initial_state()
    P0 = m * np.array([0.3, -0.2, 0.5])
    o.set_state(pos, quat, P0[None, :], phi, latch)
    n = 400
    o.step(n)
    st = o.read_state()
    assert st.linmom[0] == pytest.approx(P0 * f ** n, rel=1e-12)
    disp = dt / m * P0 * sum(f ** q for q in range(1, n + 1))
    assert st.pos[0] - pos[0] == pytest.approx(disp, rel=1e-11)


def test_ground_damping_rotational_geometric_decay():
    """The rotational analogue: M = -c_r w, c_r = 2 zeta_g sqrt(I G l^3 / 6)
    (R12: the voxel's own a2 = G J / l), I = m l^2 / 6, G = E / (2 (1 + nu)):
    phi_n = phi_0 (1 - dt c_r / I)^n; the spin axis is fixed, so the angle
    turned is dt / I * sum_{q=1..n} |phi_q| (Eq. 30)."""
    E, rho, nu, zg = 2e6, 900.0, 0.25, 0.3
    o, s = sim(np.ones((1, 1, 1)), [mat(E=E, rho=rho, nu=nu)], zeta_ground=zg)
    m = rho * L ** 3
    I = m * L * L / 6
    G = E / (2 * (1 + nu))
    cr = 2 * zg * math.sqrt(I * G * L ** 3 / 6)
    f = 1 - o.dt * cr / I
    axis = np.array([1.0, 2.0, -2.0]) / 3.0
    phi0 = I * 200.0 * axis
    pos, quat, P, phi, latch = s.initial_state()
    o.set_state(pos, quat, P, phi0[None, :], latch)
    n = 300
    o.step(n)
    st = o.read_state()
    assert st.angmom[0] == pytest.approx(phi0 * f ** n, rel=1e-12)
    turned = o.dt / I * np.linalg.norm(phi0) * sum(f ** q for q in range(1, n + 1))
    R = Rotation.from_quat(np.r_[st.quat[0, 1:], st.quat[0, 0]])
    assert R.as_rotvec() == pytest.approx(turned * axis, rel=1e-10)


# --------------------------------------------------------------- floor (R14)
@pytest.mark.parametrize("v0,zc", [(-0.05, 0.7), (0.0, 0.7), (-0.3, 0.0)])
def test_floor_first_step_normal_force(v0, zc):
    """One voxel penetrating the floor by p with vertical velocity v0, no
    gravity: the first step's normal force is F_n = max(0, k_f p - 2 zeta_col
    sqrt(m k_f) V_z) with k_f = E l (R14), so
    P_z(1) = m v0 + dt F_n exactly."""
    E, rho, p = 2e6, 1500.0, 2e-6
    o, s = sim(np.ones((1, 1, 1)), [mat(E=E, rho=rho)], floor_on=1, zeta_col=zc)
    m = rho * L ** 3
    kf = E * L
    o.set_state(np.array([[0.0, 0.0, 0.5 * L - p]]), np.array([[1.0, 0, 0, 0]]),
                np.array([[0.0, 0.0, m * v0]]), np.zeros((1, 3)), np.zeros(1, np.uint8))
    o.step(1)
    Fn = max(0.0, kf * p - 2 * zc * math.sqrt(m * kf) * v0)
    assert o.read_state().linmom[0, 2] == pytest.approx(m * v0 + o.dt * Fn, rel=1e-13)


def test_floor_normal_force_clamped_when_separating_fast():
    """A fast separating voxel: k_f p - c V_z < 0, so F_n = 0 (floors only push)."""
    E, rho, p, zc = 2e6, 1500.0, 1e-7, 1.0
    o, s = sim(np.ones((1, 1, 1)), [mat(E=E, rho=rho)], floor_on=1, zeta_col=zc)
    m = rho * L ** 3
    v0 = 0.5
    assert E * L * p - 2 * zc * math.sqrt(m * E * L) * v0 < 0
    o.set_state(np.array([[0.0, 0.0, 0.5 * L - p]]), np.array([[1.0, 0, 0, 0]]),
                np.array([[0.0, 0.0, m * v0]]), np.zeros((1, 3)), np.zeros(1, np.uint8))
    o.step(1)
    assert o.read_state().linmom[0, 2] == m * v0


# --------------------------------------------------------------- contact (R16)
def test_contact_two_materials_with_normal_damping():
    """Two voxels of different materials, lattice Manhattan 5, overlapping by q
    along x and approaching at +-u.  First step: F_on_a = max(0, k_c q - c_c
    v_n) n with n = (D_a - D_b)/|D_a - D_b| = -x, v_n = (V_a - V_b).n = -2u,
    k_c = harmonic mean of E_a l and E_b l, c_c = 2 zeta_col sqrt(m_min k_c)
    (R16)."""
    Ea, Eb, ra, rb, zc = 1e6, 5e6, 1000.0, 2000.0, 0.4
    cells = np.zeros((1, 1, 6), np.uint8)
    cells[0, 0, 0] = 1
    cells[0, 0, 5] = 2
    o, s = sim(cells, [mat(E=Ea, rho=ra), mat(E=Eb, rho=rb)], self_collision=1, zeta_col=zc)
    ma, mb = ra * L ** 3, rb * L ** 3
    pos, quat, P, phi, latch = s.initial_state()
    q, u = 0.05 * L, 0.02
    pos[1] = pos[0] + np.array([L - q, 0.0, 0.0])
    P[0, 0], P[1, 0] = ma * u, -mb * u
    o.set_state(pos, quat, P, phi, latch)
    kc = harmonic(Ea * L, Eb * L)
    cc = 2 * zc * math.sqrt(min(ma, mb) * kc)
    f = max(0.0, kc * q - cc * (-2 * u))
    o.step(1)
    st = o.read_state()
    assert st.linmom[0, 0] == pytest.approx(ma * u - o.dt * f, rel=1e-12)
    assert st.linmom[1, 0] == pytest.approx(-mb * u + o.dt * f, rel=1e-12)
    assert np.abs(st.linmom[:, 1:]).max() == 0.0


@pytest.mark.parametrize("sep,along_z", [(0.0, True), (0.5e-6, True), (2e-6, False)])
def test_contact_near_coincident_threshold(sep, along_z):
    """Reading R16: centres closer than 1e-6 l count as coincident (+-z);
    beyond that the centre line is used."""
    cells = np.zeros((1, 1, 6), np.uint8)
    cells[0, 0, 0] = 1
    cells[0, 0, 5] = 1
    o, s = sim(cells, [mat()], self_collision=1, zeta_col=0.0)
    pos, quat, P, phi, latch = s.initial_state()
    pos[1] = pos[0] + np.array([0.0, sep * L, 0.0])
    o.set_state(pos, quat, P, phi, latch)
    o.step(1)
    st = o.read_state()
    f = 1e6 * L * (L - sep * L)
    want = [0, 0, o.dt * f] if along_z else [0, -o.dt * f, 0]
    assert st.linmom[0] == pytest.approx(want, rel=1e-9, abs=1e-30)


def test_contact_coincident_centres_push_along_z():
    """Coincident centres: the normal falls back to +z for the lower
    id, -z for the other; the penalty is k_c (r_a + r_b)."""
    cells = np.zeros((1, 1, 6), np.uint8)
    cells[0, 0, 0] = 1
    cells[0, 0, 5] = 1
    o, s = sim(cells, [mat()], self_collision=1, zeta_col=0.0)
    pos, quat, P, phi, latch = s.initial_state()
    pos[1] = pos[0]
    o.set_state(pos, quat, P, phi, latch)
    o.step(1)
    st = o.read_state()
    f = 1e6 * L * L                                         # k_c (l/2 + l/2)
    assert st.linmom[0] == pytest.approx([0, 0, o.dt * f], rel=1e-12)
    assert st.linmom[1] == pytest.approx([0, 0, -o.dt * f], rel=1e-12)


# --------------------------------------------------------------- Eq. 30 (R6, R8)
@pytest.mark.parametrize("n", [1, 37, 500])
def test_free_spin_rotation_update_exact(n):
    """A free voxel spinning at constant angular momentum phi_0 (no damping,
    no bond): each step turns it by dt phi_0 / I about the fixed axis phi_0,
    applied on the left (world frame, R6), with I = m l^2 / 6 (R8).  So
    q_n = quat(n dt phi_0 / I) (x) q_0 exactly, as rotations (scipy)."""
    rho = 1700.0
    o, s = sim(np.ones((1, 1, 1)), [mat(rho=rho)])
    m = rho * L ** 3
    I = m * L * L / 6
    rng = np.random.default_rng(11)
    q0 = Rotation.from_rotvec(rng.normal(size=3))
    phi0 = I * 150.0 * rng.normal(size=3)
    pos, quat, P, phi, latch = s.initial_state()
    x, y, z, w = q0.as_quat()
    o.set_state(pos, np.array([[w, x, y, z]]), P, phi0[None, :], latch)
    o.step(n)
    st = o.read_state()
    got = Rotation.from_quat(np.r_[st.quat[0, 1:], st.quat[0, 0]])
    want = Rotation.from_rotvec(n * o.dt * phi0 / I) * q0       # left multiplication
    assert (got * want.inv()).magnitude() <= 1e-12 * max(1, n)
    # the other product order is a different rotation (the pin can tell them apart)
    other = q0 * Rotation.from_rotvec(n * o.dt * phi0 / I)
    assert (got * other.inv()).magnitude() > 1e-6
    assert np.array_equal(st.angmom[0], phi0)
    assert np.array_equal(st.pos, pos)


# --------------------------------------------------------------- Eq. 40
def test_thermal_two_material_pair_rest_length_is_mean_alpha():
    """A free two-material pair under a constant temperature offset dT relaxes
    to the separation l (1 + (alpha_a + alpha_b)/2 dT) (Eq. 40);
    alpha_a alone or alpha_b alone would give 1.1 l or 1.3 l."""
    aa, ab, dT = 0.01, 0.03, 10.0
    o, s = sim(np.array([[[1, 2]]]), [mat(cte=aa), mat(E=2e6, rho=1200.0, cte=ab)],
               zeta_bond=1.0, T_amp=dT, T_freq=0.0, T_phase=math.pi / 2)
    o.step(4000)
    st = o.read_state()
    sep = np.linalg.norm(st.pos[1] - st.pos[0])
    assert sep == pytest.approx(L * (1 + 0.5 * (aa + ab) * dT), rel=1e-9)
    assert np.abs(st.linmom).max() <= 1e-15


# --------------------------------------------------------------- friction branches (R15)
def _floor_voxel_state(o, m, pen, P=(0.0, 0.0, 0.0), latch=0):
    o.set_state(np.array([[0.0, 0.0, 0.5 * L - pen]]), np.array([[1.0, 0, 0, 0]]),
                np.array([list(P)]), np.zeros((1, 3)), np.array([latch], np.uint8))


def test_friction_breakaway_first_step():
    """A latched voxel pressed into the floor (F_n = k_f p) under a lateral force
    beyond mu_s F_n breaks away (Eq. 36 violated) and feels F_l - mu_d F_n F_l/|F_l|
    (Eq. 37, R15: opposite the applied force while V_l = 0), unlatched."""
    E, rho, p, mus, mud = 1e6, 1000.0, 2e-6, 0.6, 0.3
    o, s = sim(np.ones((1, 1, 1)), [mat(E=E, rho=rho, mu_s=mus, mu_d=mud)], floor_on=1)
    m = rho * L ** 3
    Fn = E * L * p
    Fl = np.array([0.6, -0.8]) * (1.5 * mus * Fn)          # |F_l| = 1.5 mu_s F_n
    o.set_boundary(None, np.array([[Fl[0], Fl[1], 0.0]]))
    _floor_voxel_state(o, m, p, latch=1)
    o.step(1)
    st = o.read_state()
    want = o.dt * (Fl - mud * Fn * Fl / np.linalg.norm(Fl))
    assert st.latch[0] == 0
    assert st.linmom[0, :2] == pytest.approx(want, rel=1e-12)
    # just below the threshold it stays latched and does not move laterally
    o2, _ = sim(np.ones((1, 1, 1)), [mat(E=E, rho=rho, mu_s=mus, mu_d=mud)], floor_on=1)
    o2.set_boundary(None, np.array([[0.99 * mus * Fn, 0.0, 0.0]]))
    _floor_voxel_state(o2, m, p, latch=1)
    o2.step(1)
    st2 = o2.read_state()
    assert st2.latch[0] == 1 and st2.linmom[0, 0] == 0.0 and st2.pos[0, 0] == 0.0


def test_latch_cleared_off_the_floor():
    """Out of floor contact (p <= 0) the static-friction latch is released (R15)."""
    o, s = sim(np.ones((1, 1, 1)), [mat(mu_s=0.5, mu_d=0.5)], floor_on=1)
    _floor_voxel_state(o, 1e-6, -1e-6, latch=1)             # 1 um above the floor
    o.step(1)
    assert o.read_state().latch[0] == 0


# --------------------------------------------------------------- thermal radii (R14, R16)
def test_floor_radius_swells_with_temperature():
    """A voxel resting exactly on the floor at its rest radius l/2 penetrates by
    (l/2) alpha dT once the temperature rises (contact radius of R14); with no
    gravity its first step gets P_z = dt k_f (l/2) alpha dT."""
    E, rho, a, dT = 1e6, 1000.0, 0.01, 5.0
    o, s = sim(np.ones((1, 1, 1)), [mat(E=E, rho=rho, cte=a)], floor_on=1, T_amp=dT,
               T_freq=0.0, T_phase=math.pi / 2)
    _floor_voxel_state(o, rho * L ** 3, 0.0)
    o.step(1)
    assert o.read_state().linmom[0, 2] == pytest.approx(o.dt * E * L * 0.5 * L * a * dT, rel=1e-12)


def test_contact_radius_swells_with_temperature():
    """Two voxels 1.01 l apart (no contact at rest radii) touch once dT swells
    their radii to (l/2)(1 + alpha dT): force k_c (r_a + r_b - d) (R16)."""
    aa, ab, dT = 0.02, 0.04, 1.0
    cells = np.zeros((1, 1, 6), np.uint8)
    cells[0, 0, 0] = 1
    cells[0, 0, 5] = 2
    o, s = sim(cells, [mat(cte=aa), mat(E=2e6, cte=ab)], self_collision=1, zeta_col=0.0,
               T_amp=dT, T_freq=0.0, T_phase=math.pi / 2)
    pos, quat, P, phi, latch = s.initial_state()
    d = 1.01 * L
    pos[1] = pos[0] + np.array([d, 0.0, 0.0])
    o.set_state(pos, quat, P, phi, latch)
    o.step(1)
    kc = harmonic(1e6 * L, 2e6 * L)
    q = 0.5 * L * (1 + aa * dT) + 0.5 * L * (1 + ab * dT) - d
    assert q > 0
    assert o.read_state().linmom[0, 0] == pytest.approx(-o.dt * kc * q, rel=1e-12)


# --------------------------------------------------------------- R7, R16 invariants
def test_bond_loads_invariant_under_quaternion_sign():
    """q and -q are the same orientation: flipping the sign of voxel b's (or a's)
    quaternion leaves every bond load unchanged (R7: the w >= 0 branch of the
    rotation vector of q_a* q_b)."""
    o, s = sim(np.array([[[1, 2]]]), [mat(), mat(E=3e6, rho=1500.0)], zeta_bond=0.7)
    rng = np.random.default_rng(21)
    for axis in range(3):
        qa = Rotation.from_rotvec(rng.normal(size=3) * 0.3)
        qb = Rotation.from_rotvec(qa.as_rotvec() + rng.normal(size=3) * 0.05)
        def state(q, D, P, phi):
            x, y, z, w = q.as_quat()
            return np.r_[D, w, x, y, z, P, phi]
        Da = np.zeros(3); Db = qa.apply(np.eye(3)[axis]) * L + rng.normal(size=3) * 1e-5
        sa = state(qa, Da, rng.normal(size=3) * 1e-9, rng.normal(size=3) * 1e-14)
        sb = state(qb, Db, rng.normal(size=3) * 1e-9, rng.normal(size=3) * 1e-14)
        ref = np.concatenate(o.bond_loads(0, 1, axis, sa, sb))
        for flip_a, flip_b in ((False, True), (True, False), (True, True)):
            a2, b2 = sa.copy(), sb.copy()
            if flip_a:
                a2[3:7] *= -1
            if flip_b:
                b2[3:7] *= -1
            got = np.concatenate(o.bond_loads(0, 1, axis, a2, b2))
            assert got == pytest.approx(ref, rel=1e-12, abs=1e-12 * np.abs(ref).max())


def test_interior_voxels_feel_no_contact():
    """Self collision is between surface voxels: a foreign voxel placed on
    the interior voxel of a 3x3x3 cube pushes on nothing (the centre is not a
    surface voxel, and the intruder's partners are surface voxels only), so the
    step equals the one without self collision for the cube's centre."""
    cells = np.zeros((3, 3, 8), np.uint8)
    cells[:, :, :3] = 1
    cells[1, 1, 7] = 1
    runs = []
    for col in (0, 1):
        o, s = sim(cells, [mat()], self_collision=col, zeta_col=0.0)
        pos, quat, P, phi, latch = s.initial_state()
        ijk = s.voxel_coords()
        centre = int(np.nonzero((ijk == [1, 1, 1]).all(1))[0][0])
        intruder = int(np.nonzero((ijk == [7, 1, 1]).all(1))[0][0])
        pos[intruder] = pos[centre] + np.array([0.3 * L, 0.0, 0.0])
        o.set_state(pos, quat, P, phi, latch)
        o.step(1)
        runs.append(o.read_state().linmom[centre])
    assert np.array_equal(runs[0], runs[1])
