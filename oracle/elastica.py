"""TEST INFRASTRUCTURE ONLY -- large-deflection cantilever (Euler elastica).

Closed form of the continuum problem the settled C1 cantilever approximates
("C1 as written"): a clamped inextensible Euler-Bernoulli beam
of span L with a dead tip load P perpendicular to the undeformed axis.

    EI dtheta/ds = M(s),  M(s) = P (x_tip - x(s)),   theta(0) = 0,
    equivalently  EI theta'' = -P cos(theta),  theta'(L) = 0.

Solved by shooting on theta'(0).  In the small-load limit the tip deflection
reduces to the textbook P L^3 / (3 E I) ("analytical solution").
"""
from __future__ import annotations

import numpy as np
from scipy.integrate import solve_ivp
from scipy.optimize import brentq


def linear_tip_deflection(P, L, E, I):
    """delta = P L^3 / (3 E I)."""
    return P * L ** 3 / (3.0 * E * I)


def tip_deflection(P, L, E, I):
    """Returns (vertical tip deflection, tip rotation) of the elastica."""
    EI = E * I

    def rhs(s, y):
        th, k, x, z = y
        return [k, -P / EI * np.cos(th), np.cos(th), np.sin(th)]

    def shoot(k0):
        sol = solve_ivp(rhs, (0.0, L), [0.0, k0, 0.0, 0.0], rtol=1e-12, atol=1e-15)
        return sol.y[1, -1], sol

    k_lin = P * L / EI      # linear curvature at the root
    lo, hi = 0.0, 2.0 * k_lin
    r = brentq(lambda k0: shoot(k0)[0], lo, hi, xtol=1e-16, rtol=1e-14)
    _, sol = shoot(r)
    return sol.y[3, -1], sol.y[0, -1]
