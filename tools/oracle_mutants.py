"""Mutation check of the oracle pins: apply one plausible
mistake at a time to a scratch copy of oracle/ (a dropped term, a wrong
sign, index, constant or rounding), rebuild it, and run the CPU pin tests;
every mutant must be killed (some test fails).

python tools/oracle_mutants.py [-j 4]      -> prints one line per mutant, exit 1 if any survives
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN_TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_bwd_pins.py",
             "tests/test_oracle_apx_pins.py", "tests/test_oracle_f32_tables.py"]

K = "oracle/ktanh_oracle.c"
A = "oracle/apx_oracle.c"
# (name, file, original text, mutated text)
MUTANTS = [
    ("T1 threshold", K, "static const double T1 = 0.25;", "static const double T1 = 0.2501;"),
    ("T2 threshold", K, "static const double T2 = 3.75;", "static const double T2 = 3.5;"),
    ("index: exponent bits", K, "return ((E & 3) << 3) | M_top3;", "return ((E & 1) << 3) | M_top3;"),
    ("index: mantissa bits", K, "int t = index_t(E, M >> 4);", "int t = index_t(E, M >> 3 & 7);"),
    ("line 8: sign of b", K, "int Mo = (M >> rt) + bt;", "int Mo = (M >> rt) - bt;"),
    ("line 8: shift", K, "int Mo = (M >> rt) + bt;", "int Mo = (M >> (rt + 1)) + bt;"),
    ("F32 b unit", K, "bt * (1 << (23 - pb))", "bt * (1 << (22 - pb))"),
    ("F32 index", K, "int t = index_t(E, (int)(M >> 20));", "int t = index_t(E, (int)(M >> 19) & 7);"),
    ("saturation value", K, "return (uint16_t)((s << 15) | (127 << 7) | 0);",
     "return (uint16_t)((s << 15) | (126 << 7) | 0);"),
    ("sigmoid sign", K, "return kto_bf16_encode_rne((1.0 + tv) / 2.0);",
     "return kto_bf16_encode_rne((1.0 - tv) / 2.0);"),
    ("sigmoid argument", K, "uint16_t h = kto_bf16_encode_rne(xv / 2.0);          /* x/2 in BF16 */",
     "uint16_t h = kto_bf16_encode_rne(xv / 4.0);"),
    ("swish factor", K, "return rnbf16_exact_sum(hx, hx * tv);                 /* RN_bf16(x (1+t)/2), product exact */",
     "return rnbf16_exact_sum(hx, hx * tv / 2.0);"),
    ("gelu outer: binary64 double rounding", K,
     "return rnbf16_exact_sum(hx, hx * tv);                 /* RN_bf16(x/2 (1+t)), product exact */",
     "return kto_bf16_encode_rne(xv / 2.0 * (1.0 + tv));"),
    ("bf16 exact-sum tie break", K, "return ((e > 0.0) == (gv > fv)) ? g : f;", "return f;"),
    ("gelu constant a", K, "static const double GELU_A = 0.044715;", "static const double GELU_A = 0.04715;"),
    ("gelu cubic term", K, "float p = fmaf(C1, x2, C0);", "float p = fmaf(C1, x, C0);"),
    ("bwd tanh", K, "case 0: return 1.0 - a * a;", "case 0: return 1.0 - a;"),
    ("bwd swish", K, "case 2: return (1.0 + tv) / 2.0 + a * (1.0 - tv * tv) / 4.0;",
     "case 2: return (1.0 + tv) / 2.0 + a * (1.0 - tv * tv) / 2.0;"),
    ("bf16 RNE -> truncation", K, "double nq = nearbyint(q);", "double nq = floor(q);"),
    ("optimizer: b* rounding", K, "floor_div(2 * S + ((__int128)cnt << r), (__int128)cnt << (r + 1))",
     "floor_div(2 * S, (__int128)cnt << (r + 1))"),
    ("optimizer: clip value", K, "else Mhat[j] = (1 << q) - 1;", "else Mhat[j] = (1 << q) - 2;"),
    ("optimizer: E cap", K, "int E = Ei[c] < 126 ? Ei[c] : 126;", "int E = Ei[c];"),
    ("bounds: b_max", K, "*bmax = (1 << p) - 1 - ", "*bmax = (1 << p) - "),
    ("lstm cell sum", K, "float cn = rn32_exact_sum(f * c, i * g);", "float cn = rn32_exact_sum(f * c, i * o);"),
    ("exact-sum tie break", K, "return ((e > 0.0) == ((double)g > (double)f)) ? g : f;", "return f;"),
    ("via-bf16 widening", K, "return (uint32_t)kto_ktanh_bf16(b, TE, Tr, Tb) << 16;",
     "return (uint32_t)kto_ktanh_bf16(b, TE, Tr, Tb) << 15;"),
    ("maclaurin recurrence", A, "t[k + 1] = ((k == 0 ? 1.0L : 0.0L) - conv)",
     "t[k + 1] = ((k == 0 ? 1.0L : 0.0L) + conv)"),
    ("comparator saturation", A, "#define APX_XSAT 8.0", "#define APX_XSAT 7.5"),
    ("p23 Step 1 rounding", K, "else u = bits_from_f32((float)y);", "else u = bits_from_f32((float)y) & ~1u;"),
    ("optimizer r range", K, "for (int r = 0; r <= p; ++r) {", "for (int r = 1; r <= p; ++r) {"),
    ("F32 NaN passthrough", K, "if (isnan(ax)) return x;                              /* A6 */",
     "if (isnan(ax)) return 0x7FC00000u;"),
    ("bwd sigmoid", K, "case 1: return a * (1.0 - a);", "case 1: return a * (1.0 + a);"),
    ("bwd gelu derivative", K, "c * (1.0 + 3.0 * ga * a * a);", "c * (1.0 + ga * a * a);"),
    ("taylor centre", A, "a - (k * APX_WIDTH + 0.25)", "a - (k * APX_WIDTH + 0.2)"),
    ("pade denominator order", A, "poly(par + 1, p, a) / poly(par + 2 + p, q, a)",
     "poly(par + 1, p, a) / poly(par + 2 + p, q - 1, a)"),
]


def apply(dst, f, old, new):
    p = os.path.join(dst, f)
    s = open(p).read()
    if old not in s:
        return False
    open(p, "w").write(s.replace(old, new, 1))
    return True


def run_one(m):
    name, f, old, new = m
    d = tempfile.mkdtemp(prefix="kt_mut_")
    try:
        for sub in ("oracle", "tests", "workloads"):
            shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
        if not apply(d, f, old, new):
            return name, "NOT APPLIED (pattern missing)"
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            "-m", "not gpu"] + PIN_TESTS, cwd=d, capture_output=True, text=True,
                           timeout=1800)
        if r.returncode == 0:
            return name, "SURVIVED"
        last = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED") or ln.startswith("ERROR")]
        return name, "killed by " + (last[0].split(" - ")[0] if last else f"rc={r.returncode}")
    finally:
        shutil.rmtree(d, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=4)
    ap.add_argument("-k", default="", help="only mutants whose name contains this")
    args = ap.parse_args()
    muts = [m for m in MUTANTS if args.k in m[0]]
    with ThreadPoolExecutor(args.j) as ex:
        res = list(ex.map(run_one, muts))
    bad = 0
    for name, verdict in res:
        print(f"{name:28s} {verdict}")
        bad += not verdict.startswith("killed")
    print(f"{len(res) - bad}/{len(res)} mutants killed")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
