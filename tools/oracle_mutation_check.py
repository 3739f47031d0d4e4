"""Mutation check for the oracle pins: apply plausible single mistakes to a copy of oracle/,
rebuild, run tests/test_oracle_pins.py against the mutant, and require that every mutant fails.

Usage:  python tools/oracle_mutation_check.py      (CPU only, ~2 min)
Writes profiles/oracle_mutation_check.txt.
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ALGO = "oracle/oracle_algo.inc"
MAIN = "oracle/mstrsm_oracle.c"
SCAL = "oracle/oracle_scalar.h"
GEN = "oracle/oracle_gen.inc"
PINS, GPINS = "tests/test_oracle_pins.py", "tests/test_oracle_gen.py"
INIT = "oracle/__init__.py"
SPINS, BPINS, SIDEPINS = "tests/test_oracle_spectral.py", "tests/test_oracle_backtransform.py", "tests/test_oracle_side.py"

MUTANTS = [
    ("growth bound uses cnl*|d| (eq. 5)", ALGO, "g = g * (1.0 + cnl[l] / ad);", "g = g * (1.0 + cnl[l] * ad);"),
    ("panel term dropped from G (P:392)", ALGO, "G = G + P[b] * xm;", "G = G + xm;"),
    ("precheck || instead of && (P:267)", ALGO, "if (M < OMEGA && g < OMEGA) {                  /* P:267 */",
     "if (M < OMEGA || g < OMEGA) {"),
    ("step (ii) forgets rows I0", ALGO, "for (int64_t i = 0; i < lo; i++) x[i] = LDX(x[i], -kt);          /* I0 */", ""),
    ("step (ii) forgets rows I2", ALGO, "for (int64_t i = h; i < r; i++) x[i] = LDX(x[i], -kt);           /* I2 */", ""),
    ("GEMM operand transposed (P:408)", ALGO,
     "for (int64_t i = 0; i < lo; i++) x[i] = SUB(x[i], MUL(UA(i, l), x[l]));\n    }\n    return e;",
     "for (int64_t i = 0; i < lo; i++) x[i] = SUB(x[i], MUL(UA(l, i), x[l]));\n    }\n    return e;"),
    ("op C misses the conjugate", ALGO,
     "for (int64_t i = hi; i < m; i++) x[i] = SUB(x[i], MUL(CONJ(UA(l, i)), x[l]));\n    }\n    return e;",
     "for (int64_t i = hi; i < m; i++) x[i] = SUB(x[i], MUL(UA(l, i), x[l]));\n    }\n    return e;"),
    ("complex multiply sign", SCAL, "a.re * b.im + a.im * b.re", "a.re * b.im - a.im * b.re"),
    ("Smith division sign", SCAL, "(a.im - a.re * r) / den", "(a.im + a.re * r) / den"),
    ("delta = 2^-40 ||U|| (P:231-233)", ALGO, "ldexp(unorm, -52)", "ldexp(unorm, -40)"),
    ("minpow2 not minimal", MAIN, "while (k > 1 && ldexp(a, -(k - 1)) < L) k--;", "k += 1;"),
    ("cnl not block-local", ALGO, "for (int64_t l = lo; l < k; l++) { double a = MOD(UA(l, k)); if (a > c) c = a; }",
     "for (int64_t l = 0; l < k; l++) { double a = MOD(UA(l, k)); if (a > c) c = a; }"),
    ("guarded loop keeps precheck g (P:273)", ALGO, "g = 0.0;                                    /* P:273 */", ""),
    ("guarded rescale threshold > instead of >=", ALGO, "if (g >= OMEGA) {                        /* P:301-313 */",
     "if (g > OMEGA * 2.0) {"),
    ("Lanczos drops beta v_prev", MAIN, "w[i].re = (w[i].re - a * v[i].re) - beta_prev * vp[i].re;",
     "w[i].re = (w[i].re - a * v[i].re);"),
    ("bisection returns the second-largest", MAIN, "if (sturm_below(a, b, k, mid, pivmin) == k) hi = mid; else lo = mid;",
     "if (sturm_below(a, b, k, mid, pivmin) >= k - 1) hi = mid; else lo = mid;"),
    ("TriangEig diag(Z) := 1 instead of s (P:530)", ALGO, "Z[q * ldz + k] = REAL(ldexp(1.0, e[q]));", "Z[q * ldz + k] = REAL(1.0);"),
    ("TriangEig RHS +T instead of -T (P:521)", ALGO, "Z[q * ldz + i] = i < k ? NEG(T[k * ldt + i]) : ZERO();",
     "Z[q * ldz + i] = i < k ? T[k * ldt + i] : ZERO();"),
    ("zmod prescale wrong direction", SCAL, "if (big > 0x1p+500) s = -600;", "if (big > 0x1p+500) s = 600;"),
    ("op C diag not conjugated", ALGO, "x[l] = DIV(x[l], CONJ(SUB(UA(l, l), s)));", "x[l] = DIV(x[l], SUB(UA(l, l), s));"),
    # generalized solve (Alg. 7/8) and GeneralizedTriangEig (Alg. 9), run against tests/test_oracle_gen.py
    ("gen: V update sign (P:896 += V C)", GEN, "x[i] = SUB(x[i], MUL(VA(i, l), NEG(c[l - lo])));",
     "x[i] = SUB(x[i], MUL(VA(i, l), c[l - lo]));", GPINS),
    ("gen: V update dropped", GEN, "x[i] = SUB(x[i], MUL(VA(i, l), NEG(c[l - lo])));", "(void)0;", GPINS),
    ("gen: U' without lambda (P:873)", GEN, "#define UP(i, l) SUB(UA(i, l), MUL(lam, VA(i, l)))",
     "#define UP(i, l) SUB(UA(i, l), VA(i, l))", GPINS),
    ("gen: panel term drops |lambda| ||V|| (P:952)", GEN, "G = G + (PU[b] + alam * PV[b]) * xm;",
     "G = G + PU[b] * xm;", GPINS),
    ("gen: C formed before the G(j) rescale (as printed in Alg. 8, R32)", GEN,
     [("for (int64_t l = lo; l < h; l++) c[l - lo] = MUL(lam, x[l]);\n", ""),
      ("G = G + (PU[b] + alam * PV[b]) * xm;",
       "for (int64_t l = lo; l < h; l++) c[l - lo] = MUL(lam, x[l]);\n            G = G + (PU[b] + alam * PV[b]) * xm;")],
     None, GPINS),
    ("gen: lambda = S/T (P:985)", GEN, "lam[q] = DIV(T[k * ldt + k], Sm[k * lds + k]);",
     "lam[q] = DIV(Sm[k * lds + k], T[k * ldt + k]);", GPINS),
    ("gen: Z RHS ignores S diag(lambda) (P:987)", GEN,
     "Z[q * ldz + i] = i < k ? SUB(MUL(Sm[k * lds + i], lam[q]), T[k * ldt + i]) : ZERO();",
     "Z[q * ldz + i] = i < k ? NEG(T[k * ldt + i]) : ZERO();", GPINS),
    # SURVEY §8f f2-f4 (Python / C oracle parts), each against its own pin file
    ("cloud: absolute instead of relative settle test (R33)", MAIN, "fabs(theta - theta_prev) <= J->tol * theta",
     "fabs(theta - theta_prev) <= J->tol", SPINS),
    ("cloud: previous Ritz value never updated (R33)", MAIN, "                theta_prev = theta;\n", "", SPINS),
    ("portrait: pad 0.5 instead of 0.25 (R34)", INIT, "pad = 0.25 * max(", "pad = 0.5 * max(", SPINS),
    ("window: grid index iy + ny ix (R15)", INIT, "return (gx[None, :] + 1j * gy[:, None]).reshape(-1)",
     "return (gx[:, None] + 1j * gy[None, :]).reshape(-1)", SPINS),
    ("backtransform: Q^T Z (P:540)", INIT, "return np.asfortranarray(np.asarray(Q) @ np.asarray(Z))",
     "return np.asfortranarray(np.asarray(Q).T @ np.asarray(Z))", BPINS),
    ("side L,L: shifts not conjugated", INIT, 'return mstrsm(np.triu(cj(A.T)), cj(s), B, op="C"',
     'return mstrsm(np.triu(cj(A.T)), s, B, op="C"', SIDEPINS),
    ("side R,U: A not conjugated", INIT, 'X, e = mstrsm(np.triu(cj(A)), cj(s), B.T, op="C"',
     'X, e = mstrsm(np.triu(A), cj(s), B.T, op="C"', SIDEPINS),
    ("side R,L: A instead of A^T", INIT, 'X, e = mstrsm(np.triu(A.T), s, B.T, op="N"',
     'X, e = mstrsm(np.triu(A), s, B.T, op="N"', SIDEPINS),
]


def main():
    lines = []
    survived = 0
    for mut in MUTANTS:
        name, rel, old, new = mut[:4]
        tests = mut[4] if len(mut) > 4 else PINS
        tmp = tempfile.mkdtemp(prefix="omut_")
        try:
            for d in ("oracle", "tests", "paper_1607_01477_b200"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__", "*.o"))
            p = os.path.join(tmp, rel)
            src = open(p).read()
            for o, n in (old if isinstance(old, list) else [(old, new)]):
                if o not in src:
                    raise SystemExit(f"mutation site not found: {name}")
                src = src.replace(o, n, 1)
            open(p, "w").write(src)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                                tests], cwd=tmp, capture_output=True, text=True,
                               timeout=600)
            killed = r.returncode != 0
            first = next((ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")), "")
            lines.append(f"{'KILLED ' if killed else 'SURVIVED'}  {name}  {first[:110]}")
            survived += not killed
            print(lines[-1], flush=True)
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
    lines.append(f"{len(MUTANTS) - survived}/{len(MUTANTS)} mutants killed")
    print(lines[-1])
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", "oracle_mutation_check.txt"), "w").write("\n".join(lines) + "\n")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
