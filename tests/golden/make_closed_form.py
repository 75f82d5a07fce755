"""Writes tests/golden/config1_closed_form.json: closed-form values for
BASELINE.json config 1 (Dirichlet-CC 64x64, h = 1/64, λ = h²/8 = 2^-15, φ0 = 0,
ρ = sin πx sin πy at cell centres).  Uses mpmath only -- no oracle, no GPU.

ρ is the (1,1) eigenvector of Δ_h with μ = -(8/h²) sin²(πh/2); one Jacobi sweep
(Eq.3) maps φ -> g φ - λρ with g = 1 + λμ = cos²(π/128), so
φ^n = (1 - g^n) ρ/μ and r(φ^n) = -g^n ρ; max|ρ| = sin²(31.5π/64) = g.
"""
import json
import os

import mpmath as mp

mp.mp.dps = 40
n = 64
h = mp.mpf(1) / n
lam = mp.mpf(2) ** -15
mu = -8 / h**2 * mp.sin(mp.pi * h / 2) ** 2
g = 1 + lam * mu
g_check = mp.cos(mp.pi / 128) ** 2
assert abs(g - g_check) < mp.mpf(10) ** -35
rhomax = mp.sin(mp.pi * (31 + mp.mpf(1) / 2) / 64) ** 2
lam1 = mp.mpf(2) ** -14
g1 = 1 + lam1 * mu
out = {
    "_doc": __doc__,
    "g": float(g),
    "mu11": float(mu),
    "resmax_phi99": float(g**99 * rhomax),
    "resmax_phi100": float(g**100 * rhomax),
    "max_phi100": float((1 - g**100) * rhomax / abs(mu)),
    "max_phi100_omega1": float((1 - g1**100) * rhomax / abs(mu)),
    "l2h_phi_k": "g**k / 2",
}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "config1_closed_form.json"), "w") as f:
    json.dump(out, f, indent=2)
print(out)
