"""Mutation check of the GPU parity tests: one plausible mistake at a time in
a scratch copy of the CUDA sources, built into its own libktanh.so; the GPU
parity tests, run against each mutant through KT_LIB, must fail.

  python tools/kernel_mutants.py build [-j 4]   # here (nvcc cross-compiles): abtmp/mut_*.so
  python tools/kernel_mutants.py run            # on the GPU box: one line per mutant
"""
import argparse
import glob
import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "abtmp")
D = "kt_device.cuh"
KK = "kt_kernels.cu"
G = "kt_gemm.cu"
API = "kt_api.cu"
APX = "kt_apx.cu"
# (name, file under csrc/, original text, mutated text, tests that must catch it)
PARITY = "tests/test_gpu_parity.py"
MUTANTS = [
    ("bf16 T1 threshold", D, "constexpr uint32_t kT1x2 = 0x3E803E80u;",
     "constexpr uint32_t kT1x2 = 0x3E813E81u;", PARITY),
    ("f32 saturate at T2", D, "uint32_t y = (u2 > (kT2f << 1)) ? 0x3F800000u : ym;",
     "uint32_t y = (u2 >= (kT2f << 1)) ? 0x3F800000u : ym;", PARITY),
    ("sigmoid outer constant", D, "  return hfma2_bf16(t, kHalfx2, kHalfx2);",
     "  return hfma2_bf16(t, kHalfx2, 0x3F013F01u);", PARITY),
    ("gelu C1 one ulp", D, "constexpr uint32_t kGeluC1Bits = 0x3D122279u;",
     "constexpr uint32_t kGeluC1Bits = 0x3D12227Au;", PARITY),
    ("gelu bwd C3", D, "constexpr uint32_t kGeluC3Bits = 0x3DDB33B6u;",
     "constexpr uint32_t kGeluC3Bits = 0x3DDB43B6u;", "tests/test_gpu_bwd.py"),
    ("ragged tail off by one", KK, "scalar_span<OP, FMT>(x + toff, y + toff, tail, L);",
     "scalar_span<OP, FMT>(x + toff, y + toff, tail ? tail - 1 : 0, L);", PARITY),
    ("lstm cell double rounding", D, "return pack_bf16x2(mul_rodd(ov.y, th), mul_rodd(ov.x, tl));",
     "return pack_bf16x2(ov.y * th, ov.x * tl);", PARITY),
    ("via-bf16 rounding", D, "const uint32_t b = pack_bf16x2(0.0f, __uint_as_float(u));",
     "const uint32_t b = u >> 16;", PARITY),
    ("64-entry half select", D, "const uint32_t Ll = (x & 0x100u) ? l1 : l0;",
     "const uint32_t Ll = (x & 0x80u) ? l1 : l0;", PARITY),
    ("gemm epilogue column order", G,
     "w0[j] = pack_bf16x2(__uint_as_float(r[2 * j + 1]), __uint_as_float(r[2 * j]));",
     "w0[j] = pack_bf16x2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));",
     "tests/test_gpu_gemm.py"),
    ("gemm cell gate order", G,
     "const uint32_t gf = pack_bf16x2(__uint_as_float(r[8 + 2 * k + 1]), __uint_as_float(r[8 + 2 * k]));",
     "const uint32_t gf = pack_bf16x2(__uint_as_float(r[24 + 2 * k + 1]), __uint_as_float(r[24 + 2 * k]));",
     "tests/test_gpu_gemm.py"),
    ("p = 23 table word", API,
     "((int64_t)E[t] << 23) + (int64_t)b[t] - ((int64_t)e_in(t) << (23 - r[t]));",
     "((int64_t)E[t] << 23) + (int64_t)b[t] + 1 - ((int64_t)e_in(t) << (23 - r[t]));",
     "tests/test_gpu_f32_tables.py"),
    ("pair GEMM B rank offset", G, "(int)(nb * 256 + rank * Sh::kBRows)", "(int)(nb * 256)",
     "tests/test_gpu_gemm.py"),
    ("f32 inf takes bypass", D, "const bool byp = (u2 - (kT1f << 1)) > ((kInff << 1) - (kT1f << 1));",
     "const bool byp = (u2 - (kT1f << 1)) >= ((kInff << 1) - (kT1f << 1));", PARITY),
    ("swish bwd factor", D, "return fma2(mul2(hx, half), fma2(neg2(t), t, splat2(1.0f)), fma2(t, half, half));",
     "return fma2(hx, fma2(neg2(t), t, splat2(1.0f)), fma2(t, half, half));", "tests/test_gpu_bwd.py"),
    ("dual kernel output swap", KK, "    st256(ys + hb + i * kVecBytes, sw, i < nvec);",
     "    st256(ys + hb + i * kVecBytes, g, i < nvec);", PARITY),
    ("taylor comparator centre", APX, "h = __fsub_rn(h, k != 0 ? 0.25f : 0.0f);",
     "h = __fsub_rn(h, k != 0 ? 0.2f : 0.0f);", "tests/test_gpu_apx.py"),
    ("pade comparator saturation", APX, "return a >= w.xsat ? 1.0f : y;", "return a > 2.0f * w.xsat ? 1.0f : y;",
     "tests/test_gpu_apx.py"),
    # round 2: the exact outer step (R-DERIVED) and the per-kernel unroll
    ("tie patch direction", D, "      const uint32_t inc = (s == 0 && (OP == OP_GELU || m >= 2)) ? 1u : 0u;",
     "      const uint32_t inc = (s != 0 && (OP == OP_GELU || m >= 2)) ? 1u : 0u;", PARITY),
    ("f32 tie patch direction", D, "\n  const uint32_t inc = (s == 0 && (OP == OP_GELU || m >= 2)) ? 1u : 0u;",
     "\n  const uint32_t inc = (s != 0 && (OP == OP_GELU || m >= 2)) ? 1u : 0u;", PARITY),
    ("tie screen threshold", D, "return (kmin & 0xFF00u) == 0 || (kmin & 0xFF000000u) == 0;",
     "return (kmin & 0xFF80u) == 0 || (kmin & 0xFF800000u) == 0;", PARITY),
    ("outer_exact rounds both ways", D,
     "const uint32_t up = hset2_gt(r, 0u) & hset2_ne(t, 0u) & kOnex2;     // 1.0 where the t-term rounds up",
     "const uint32_t up = hset2_ne(r, 0u) & hset2_ne(t, 0u) & kOnex2;", PARITY),
    ("f32 outer tie ignored", D, "const float c = (r > 0.0f && t != 0.0f) ? __fadd_rn(hx, r) : hx;",
     "const float c = hx;", PARITY),
    ("f32 tie screen threshold", D, "constexpr uint32_t kTieKeyF32 = 0x01000000u << 1;",
     "constexpr uint32_t kTieKeyF32 = 0x00800000u << 1;", PARITY),
    ("dual tie fix-up dropped", KK, "    tie_fixup_dual<FMT, U>(x + hb, yg + hb, ys + hb, base, nvec);   // rare",
     "    (void)0;", PARITY),
    ("map grid for a larger chunk", KK,
     "  const uint64_t nchunks = (nvec + 32 * U - 1) / (32 * U);\n  if (nchunks / kW >= 0x7FFFFFFFull)",
     "  const uint64_t nchunks = (nvec + 64 * U - 1) / (64 * U);\n  if (nchunks / kW >= 0x7FFFFFFFull)", PARITY),
    ("host pipeline chunk offset", API,
     "KT_CK(cudaMemcpyAsync(yh + off * es, dy, cnt * es, cudaMemcpyDeviceToHost, d2h), \"D2H\");",
     "KT_CK(cudaMemcpyAsync(yh + off * es, dy, (cnt - (cnt > 1)) * es, cudaMemcpyDeviceToHost, d2h), \"D2H\");",
     PARITY),
]


def slug(name):
    return "".join(c if c.isalnum() else "_" for c in name)


def build_one(m):
    name, f, old, new, _ = m
    sys.path.insert(0, os.path.join(ROOT, "paper_1909_07729_b200"))
    import build as B
    d = tempfile.mkdtemp(prefix="kt_kmut_")
    try:
        csrc = os.path.join(d, "csrc")
        shutil.copytree(B.CSRC, csrc)
        p = os.path.join(csrc, f)
        s = open(p).read()
        if s.count(old) != 1:
            return name, f"NOT APPLIED ({s.count(old)} matches)"
        open(p, "w").write(s.replace(old, new))
        out = os.path.join(OUT, f"mut_{slug(name)}.so")
        flags = [x for x in B.NVCC_FLAGS if x not in ("-Xptxas", "-v")]
        cmd = ["nvcc"] + flags + ["-I", B.INCLUDE, "-I", csrc, "-o", out] + \
            sorted(glob.glob(os.path.join(csrc, "*.cu")))
        r = subprocess.run(cmd, capture_output=True, text=True)
        return name, "built" if r.returncode == 0 else "BUILD FAILED: " + r.stderr[-300:]
    finally:
        shutil.rmtree(d, ignore_errors=True)


def run_one(m):
    name, _, _, _, tests = m
    so = os.path.join(OUT, f"mut_{slug(name)}.so")
    if not os.path.exists(so):
        return name, "MISSING .so"
    env = dict(os.environ, KT_LIB=so)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                        tests], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    if r.returncode == 0:
        return name, "SURVIVED"
    failed = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED") or ln.startswith("ERROR")]
    return name, "killed by " + (failed[0].split(" - ")[0] if failed else f"rc={r.returncode}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["build", "run"])
    ap.add_argument("-j", type=int, default=4)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    if args.mode == "build":
        with ThreadPoolExecutor(args.j) as ex:
            res = list(ex.map(build_one, MUTANTS))
    else:
        res = [run_one(m) for m in MUTANTS]
    bad = 0
    for name, verdict in res:
        print(f"{name:30s} {verdict}", flush=True)
        bad += args.mode == "run" and not verdict.startswith("killed")
    if args.mode == "run":
        print(f"{len(res) - bad}/{len(res)} mutants killed")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
