"""Mutation check of the oracle pins: apply plausible single mistakes to
oracle/protox_oracle.cpp (dropped term, wrong sign, wrong index, swapped
operand, wrong order), rebuild into /tmp, and confirm that
tests/test_oracle_pins.py fails for every mutant.  CPU only.

    python scripts/oracle_mutation_check.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "protox_oracle.cpp")

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


def main():
    src = open(SRC).read()
    survivors = []
    for name, old, new in MUTANTS:
        assert old in src, f"mutation anchor not found: {name}"
        mut = src.replace(old, new, 1)
        path = f"/tmp/orc_mut_{abs(hash(name))}.cpp"
        lib = path[:-4] + ".so"
        open(path, "w").write(mut)
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-fPIC", "-shared", path, "-o", lib])
        env = dict(os.environ, PROTOX_ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            os.path.join(ROOT, "tests", "test_oracle_pins.py")],
                           env=env, capture_output=True, text=True, cwd=ROOT)
        killed = r.returncode != 0
        first = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
        print(f"{'KILLED ' if killed else 'SURVIVED'} {name:45s} {first[0] if first else ''}")
        if not killed:
            survivors.append(name)
    print(f"{len(MUTANTS) - len(survivors)}/{len(MUTANTS)} mutants killed")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
