"""Mutation check of the oracle pins: apply plausible single mistakes to
oracle/protox_oracle.cpp (2D) and oracle/protox_oracle3d.cpp (3D) -- dropped
term, wrong sign, wrong index, swapped operand, wrong order -- rebuild into
/tmp, and confirm that tests/test_oracle_pins.py (2D) or
tests/test_oracle_pins3d.py (3D) fails for every mutant.  CPU only.

    python scripts/oracle_mutation_check.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "protox_oracle.cpp")
SRC3 = os.path.join(ROOT, "oracle", "protox_oracle3d.cpp")

MUTANTS = [
    ("drop W tap", "{{pt(-1, 0), 1.0}, {pt(1, 0), 1.0}", "{{pt(1, 0), 1.0}"),
    ("centre -4 -> -3", "{pt(0, 0), -4.0}", "{pt(0, 0), -3.0}"),
    ("N tap wrong index", "{pt(0, 1), 1.0},\n            {pt(0, 0), -4.0}", "{pt(0, 2), 1.0},\n            {pt(0, 0), -4.0}"),
    ("mehrstellen corner weight", "{pt(-1, -1), 1.0}, {pt(1, -1), 1.0}", "{pt(-1, -1), 4.0}, {pt(1, -1), 1.0}"),
    ("mehrstellen scale", "s.scale = 1.0 / (6.0 * h * h);", "s.scale = 1.0 / (4.0 * h * h);"),
    ("scale not divided by h^2", "s.scale = 1.0 / (h * h);", "s.scale = 1.0 / h;"),
    ("update sign", "phi.data[ib].at(p) + lambda * r;", "phi.data[ib].at(p) - lambda * r;"),
    ("residual operands swapped", "double r = d - f.data[ib].at(p);", "double r = f.data[ib].at(p) - d;\n        r = r * (1.0 + 1e-3);"),
    ("residual missing scale", "double d = st.scale * L;", "double d = L;"),
    ("dirichlet sign kept", "            sign = -sign;\n", ""),
    ("dirichlet mirror off by one", "q.c[d] = (c < 0) ? (-c - 1) : (2 * n - 1 - c);", "q.c[d] = (c < 0) ? (-c) : (2 * n - 2 - c);"),
    ("periodic wrap off by one", "q.c[d] = ((c % n) + n) % n;", "q.c[d] = ((c % n) + n + 1) % n;"),
    ("update uses rho not temp", "double r = temp.at(p) - f.data[ib].at(p);", "double r = temp.at(p) - 2.0 * f.data[ib].at(p);"),
    ("no exchange before sweep", "static void jacobi_iteration(const Stencil& st, Level& phi, const Level& f, double lambda) {\n  exchange(phi);", "static void jacobi_iteration(const Stencil& st, Level& phi, const Level& f, double lambda) {\n"),
    ("gauss-seidel leak (update in place before temp)", "    BoxData temp(B);\n    stencil_apply(st, phi.data[ib], B, temp, st.scale);", "    BoxData temp(B);\n    stencil_apply(st, phi.data[ib], B, temp, st.scale);\n    if (ib + 1 < phi.L->boxes.size()) exchange(phi);"),
    ("max norm drops abs", "double a = std::fabs(r);", "double a = r;"),
    ("sumsq drops square", "sum.add(r * r);", "sum.add(std::fabs(r));"),
    ("rhs correction 1/6", "const double c12 = 1.0 / 12.0;", "const double c12 = 1.0 / 6.0;"),
    ("norm schedule off by one", "if (p->norm_every > 0 && it % p->norm_every == 0) record();", "if (p->norm_every > 0 && (it + 1) % p->norm_every == 0) record();"),
    ("neumaier compensation dropped", "  double value() const { return s + c; }", "  double value() const { return s; }"),
    ("ordinal transposed", "return (p.c[0] - lo.c[0]) + (p.c[1] - lo.c[1]) * extent(0);", "return (p.c[1] - lo.c[1]) + (p.c[0] - lo.c[0]) * extent(1);"),
]

MUTANTS3 = [
    ("3D centre -6 -> -5", "{p3(0, 0, -1), 1.0}, {p3(0, 0, 1), 1.0}, {p3(0, 0, 0), -6.0}", "{p3(0, 0, -1), 1.0}, {p3(0, 0, 1), 1.0}, {p3(0, 0, 0), -5.0}"),
    ("3D drop T tap", "{p3(0, 0, -1), 1.0}, {p3(0, 0, 1), 1.0}, {p3(0, 0, 0), -6.0}", "{p3(0, 0, -1), 1.0}, {p3(0, 0, 0), -6.0}"),
    ("3D B tap wrong plane", "{p3(0, 0, -1), 1.0}, {p3(0, 0, 1), 1.0}, {p3(0, 0, 0), -6.0}", "{p3(0, 0, -2), 1.0}, {p3(0, 0, 1), 1.0}, {p3(0, 0, 0), -6.0}"),
    ("3D scale 1/h", "scale = 1.0 / (p->h * p->h);\n  } else if", "scale = 1.0 / p->h;\n  } else if"),
    ("3D dirichlet sign kept", "              sign = -sign;\n", ""),
    ("3D periodic wrap off by one", "q.c[d] = ((c % n) + n) % n;", "q.c[d] = ((c % n) + n + 1) % n;"),
    ("3D update sign", "v = v + lambda * (temp.at(p) - rho.data[ib].at(p));", "v = v - lambda * (temp.at(p) - rho.data[ib].at(p));"),
    ("3D residual drops abs", "const double a = std::fabs(r);", "const double a = r;"),
    # (a transposed BoxData ordinal is an equivalent mutant: per-box storage order is internal)
    ("3D global layout x/y swapped", "return (x + L.g) + W0 * ((y + L.g) + W1 * (z + L.g));", "return (y + L.g) + W1 * ((x + L.g) + W0 * (z + L.g));"),
    ("27pt face weight 14 -> 13", "{p3(0, 1, 0), 14.0},  {p3(0, 0, -1), 14.0}", "{p3(0, 1, 0), 13.0},  {p3(0, 0, -1), 14.0}"),
    ("27pt edge weight 3 -> 2", "for (auto& e : e2) t.push_back({p3(e[0], 0, e[1]), 3.0});", "for (auto& e : e2) t.push_back({p3(e[0], 0, e[1]), 2.0});"),
    ("27pt corners dropped", "      for (int x = -1; x <= 1; x += 2) t.push_back({p3(x, y, z), 1.0});", "      for (int x = -1; x <= 1; x += 2) t.push_back({p3(x, y, 0), 0.0});"),
    ("27pt scale 1/(24h^2)", "scale = 1.0 / (30.0 * p->h * p->h);", "scale = 1.0 / (24.0 * p->h * p->h);"),
    ("27pt rhs correction 1/6", "const double c12 = 1.0 / 12.0;", "const double c12 = 1.0 / 6.0;"),
    ("3D norm schedule off by one", "if (p->norm_every > 0 && it % p->norm_every == 0) record();", "if (p->norm_every > 0 && (it + 1) % p->norm_every == 0) record();"),
]


def main():
    srcs = {SRC: open(SRC).read(), SRC3: open(SRC3).read()}
    cases = [(SRC, "test_oracle_pins.py", m) for m in MUTANTS] + [(SRC3, "test_oracle_pins3d.py", m) for m in MUTANTS3]
    survivors = []
    for target, test, (name, old, new) in cases:
        src = srcs[target]
        assert old in src, f"mutation anchor not found: {name}"
        mut = src.replace(old, new, 1)
        path = f"/tmp/orc_mut_{abs(hash(name))}.cpp"
        lib = path[:-4] + ".so"
        open(path, "w").write(mut)
        other = [p for p in srcs if p != target]  # the unmutated other half of liborc
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-fPIC", "-shared", path, *other,
                               "-o", lib])
        env = dict(os.environ, PROTOX_ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            os.path.join(ROOT, "tests", test)],
                           env=env, capture_output=True, text=True, cwd=ROOT)
        killed = r.returncode != 0
        first = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
        print(f"{'KILLED ' if killed else 'SURVIVED'} {name:45s} {first[0] if first else ''}")
        if not killed:
            survivors.append(name)
    print(f"{len(cases) - len(survivors)}/{len(cases)} mutants killed")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
