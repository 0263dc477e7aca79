"""Mutation test of the oracle pins (CPU only).

Each mutant is oracle.cpp with one plausible one-symbol mistake in a term the
paper defines (a dropped factor, a wrong mass, a swapped product order, ...).
For every mutant the script builds a shared library under /tmp, points the
oracle package at it (VX_ORACLE_LIB) and runs the `-m "not gpu"` pin files;
a pin set is adequate for a term when at least one pin fails on its mutant.

    python tools/oracle_mutants.py > tests/oracle_mutants.txt
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.cpp")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_pins_damping.py"]

# (term, passage, old, new)
MUTANTS = [
    ("c_t factor 2 dropped", "Eq. 34",
     "double ct = 2 * zeta_bond * std::sqrt(c.m_min * c.a1);",
     "double ct = zeta_bond * std::sqrt(c.m_min * c.a1);"),
    ("c_t with m_max", "Eq. 34, R10",
     "c.m_min = std::min(ma.m, mb.m);", "c.m_min = std::max(ma.m, mb.m);"),
    ("c_r with k_phi = 2 b3 (SPEC) instead of a2", "Eq. 35, R11",
     "double cr = 2 * zeta_bond * std::sqrt(c.I_min * c.a2);",
     "double cr = 2 * zeta_bond * std::sqrt(c.I_min * 2 * c.b3);"),
    ("c_r with I_max", "Eq. 35, R10",
     "c.I_min = std::min(ma.I, mb.I);", "c.I_min = std::max(ma.I, mb.I);"),
    ("V_r cross term with r instead of r/2", "Eq. 33",
     "cross(0.5 * r, wavg)", "cross(r, wavg)"),
    ("V_r against V_a instead of the average", "Eq. 33",
     "Vec3 Vr = (VB - Vavg)", "Vec3 Vr = (VB - VA)"),
    ("bond damping sign flipped", "Eq. 34",
     "Fa = Fa + ct * Vr;", "Fa = Fa - ct * Vr;"),
    ("ground damping factor 2 dropped", "P:254, R12",
     "double cgt = 2 * env.zeta_ground * std::sqrt(M.m * M.E * l);",
     "double cgt = env.zeta_ground * std::sqrt(M.m * M.E * l);"),
    ("rotational ground damping with G l^3 (no /6)", "P:254, R12",
     "std::sqrt(M.I * M.G * l * l * l / 6.0)", "std::sqrt(M.I * M.G * l * l * l)"),
    ("inertia m l^2 / 12", "R8",
     "M.I = M.m * l * l / 6.0;", "M.I = M.m * l * l / 12.0;"),
    ("rotation update q (x) dq", "Eq. 30, R6",
     "y.q = qnormalize(qmul(dq, x.q));", "y.q = qnormalize(qmul(x.q, dq));"),
    ("rotation increment with phi_n (explicit) instead of phi_n+1", "Eq. 30",
     "Vec3 th = (dt / M.I) * y.phi;", "Vec3 th = (dt / M.I) * x.phi;"),
    ("rotation increment half angle", "Eq. 30, R6",
     "dq.w = std::cos(0.5 * a);", "dq.w = std::cos(a);"),
    ("thermal rest length with alpha_a only", "Eq. 40",
     "c.alpha_mean = 0.5 * (ma.cte + mb.cte);", "c.alpha_mean = ma.cte;"),
    ("thermal rest length with alpha sum", "Eq. 40",
     "c.alpha_mean = 0.5 * (ma.cte + mb.cte);", "c.alpha_mean = (ma.cte + mb.cte);"),
    ("floor normal damping without m", "P:274, R14",
     "double cf = 2 * env.zeta_col * std::sqrt(M.m * kf);",
     "double cf = 2 * env.zeta_col * std::sqrt(kf);"),
    ("floor force not clamped at 0", "R14",
     "if (Fn < 0) Fn = 0;", ""),
    ("contact stiffness arithmetic mean", "R16",
     "double kc = 2 * ka * kb / (ka + kb);", "double kc = 0.5 * (ka + kb);"),
    ("contact damping with m_max", "R16",
     "std::sqrt(std::min(ma.m, mb.m) * kc)", "std::sqrt(std::max(ma.m, mb.m) * kc)"),
    ("contact coincident normal sign", "S:322",
     "n = v3(0, 0, a < b ? 1.0 : -1.0);", "n = v3(0, 0, a < b ? -1.0 : 1.0);"),
    ("F_z1 sign as printed (P:194)", "Eq. 15, R1",
     "c.b1 * Z2 + c.b2 * ty", "c.b1 * Z2 - c.b2 * ty"),
    ("M_b bending 2 b3 -> b3", "Eq. 23",
     "-c.b2 * Z2 - 2 * c.b3 * ty", "-c.b2 * Z2 - c.b3 * ty"),
    ("frame of a transposed (R instead of R^T)", "P:189",
     "Vec3 d = perm_to_bond(axis, mulT(Ra, r));", "Vec3 d = perm_to_bond(axis, mul(Ra, r));"),
    ("y-bond permutation swapped", "R5",
     "if (axis == 1) return v3(a.y, a.z, a.x);", "if (axis == 1) return v3(a.y, a.x, a.z);"),
    ("dt without 2 pi", "Eq. 31",
     "env->dt_safety / (2 * kPi * std::sqrt(w2max))", "env->dt_safety / std::sqrt(w2max)"),
    ("dt with m_max", "Eq. 32",
     "w2max = std::max(w2max, B.c.a1 / B.c.m_min);",
     "w2max = std::max(w2max, B.c.a1 / std::max(s->mats[s->vox[B.a].mat].m, s->mats[s->vox[B.b].mat].m));"),
    ("position update with P_n (explicit Euler)", "Eq. 28",
     "y.D = x.D + (dt / M.m) * y.P;", "y.D = x.D + (dt / M.m) * x.P;"),
    ("gravity sign", "P:260",
     "F.z = F.z - M.m * env.gravity;", "F.z = F.z + M.m * env.gravity;"),
    ("friction halt threshold without dt", "Eq. 38",
     "if (Vl <= M.mu_d * Fn * dt / M.m)", "if (Vl <= M.mu_d * Fn / M.m)"),
    ("static friction with mu_d", "Eq. 36",
     "if (Fl <= M.mu_s * Fn)", "if (Fl <= M.mu_d * Fn)"),
    ("composite E arithmetic mean", "Eq. 1",
     "Ec = 2 * m1.E * m2.E / (m1.E + m2.E);", "Ec = 0.5 * (m1.E + m2.E);"),
    ("torsion constant J = l^4/12", "Eq. 5",
     "double J = l * l * l * l / 6.0;", "double J = l * l * l * l / 12.0;"),
    ("contact Manhattan exclusion <= 2", "P:280",
     "if (manhattan(vx, s->vox[p]) <= 3) continue;", "if (manhattan(vx, s->vox[p]) <= 2) continue;"),
    ("breakaway friction along +F_l", "Eq. 37, R15",
     "F.x = Flx - M.mu_d * Fn * Flx / Fl;", "F.x = Flx + M.mu_d * Fn * Flx / Fl;"),
    ("breakaway with mu_s", "Eq. 37, R15",
     "F.y = Fly - M.mu_d * Fn * Fly / Fl;", "F.y = Fly - M.mu_s * Fn * Fly / Fl;"),
    ("sliding friction without the F_n factor", "Eq. 37",
     "F.x = Flx - M.mu_d * Fn * V.x / Vl;", "F.x = Flx - M.mu_d * V.x / Vl;"),
    ("latch kept when leaving the floor", "R15",
     "      } else {\n        latch = false;\n      }\n    }\n    /* Eq. 27-30 (R6) */", "      }\n    }\n    /* Eq. 27-30 (R6) */"),
    ("ground damping on velocity of the wrong sign", "P:254",
     "F = F - cgt * V;", "F = F + cgt * V;"),
    ("thermal floor radius without alpha", "R14",
     "double rv = 0.5 * l * (1.0 + M.cte * dT);", "double rv = 0.5 * l;"),
    ("contact radius without thermal swell", "R16",
     "double ra = 0.5 * s->l * (1.0 + ma.cte * dT);\n  double rb", "double ra = 0.5 * s->l;\n  double rb"),
    ("rotation vector without the factor 2", "R7",
     "th = (2.0 * std::atan2(vn, qrel.w) / vn) * vq;", "th = (std::atan2(vn, qrel.w) / vn) * vq;"),
    ("no w >= 0 fold of q_rel", "R7",
     "if (qrel.w < 0) { qrel.w = -qrel.w; qrel.x = -qrel.x; qrel.y = -qrel.y; qrel.z = -qrel.z; }", ""),
    ("contact for interior voxels too", "P:278",
     "if (env.self_collision && vx.surface) {", "if (env.self_collision) {"),
    ("temperature phase dropped", "P:293",
     "std::sin(2 * kPi * s->env.T_freq * t + s->env.T_phase)", "std::sin(2 * kPi * s->env.T_freq * t)"),
]


def build(src_text, out):
    with tempfile.NamedTemporaryFile("w", suffix=".cpp", delete=False) as f:
        f.write(src_text)
        path = f.name
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                    "-shared", "-fPIC", "-I", os.path.join(ROOT, "oracle"), "-o", out, path],
                   check=True)
    os.unlink(path)


def run_pins(lib):
    env = dict(os.environ, VX_ORACLE_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", *PINS, "-q", "-p", "no:cacheprovider",
                        "-m", "not gpu and not slow", "--timeout", "900"],
                       cwd=ROOT, env=env, capture_output=True, text=True)
    failed = [ln.split(" ")[1].split("::")[-1] for ln in r.stdout.splitlines()
              if ln.startswith("FAILED ")]
    return r.returncode, failed


def main():
    base = open(SRC).read()
    print("# oracle mutation test: one plausible slip per row; 'caught by' = pins that fail")
    print(f"# pins: {', '.join(PINS)}")
    rc, failed = run_pins(os.path.join(ROOT, "oracle", "liboracle.so"))
    print(f"unmutated oracle: rc={rc} failed={failed}")
    missed = 0
    only = sys.argv[1] if len(sys.argv) > 1 else None
    todo = [m for m in MUTANTS if not only or only in m[0]]
    for term, cite, old, new in todo:
        if base.count(old) != 1:
            print(f"{term} [{cite}]: PATTERN NOT FOUND ({base.count(old)} hits)")
            missed += 1
            continue
        lib = os.path.join(tempfile.gettempdir(), "orc_mutant.so")
        build(base.replace(old, new), lib)
        rc, failed = run_pins(lib)
        caught = rc != 0
        missed += 0 if caught else 1
        print(f"{term} [{cite}]: {'caught by ' + ', '.join(failed[:4]) + (' ...' if len(failed) > 4 else '') if caught else 'NOT CAUGHT'}",
              flush=True)
    print(f"# {len(todo) - missed} / {len(todo)} mutants caught")
    return 1 if missed else 0


if __name__ == "__main__":
    sys.exit(main())
