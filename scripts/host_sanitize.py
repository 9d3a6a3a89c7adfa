#!/usr/bin/env python
"""AddressSanitizer + UndefinedBehaviorSanitizer on the HOST code:

  1. the C oracle (oracle/gsb_oracle.c) built with -fsanitize=address,undefined, driven by the
     oracle pins and the oracle-side LiDAR / blur / synth tests (CPU);
  2. libgsb's host runtime (every .cu translation unit's host code: argument validation, the
     template build, reservation, the chunked pipeline's host logic) built with
     -Xcompiler -fsanitize=address,undefined, driven by tests/test_abi.py on CPU and — when a GPU
     is visible — by a set of -m gpu tests (renders, static pre-binning, LiDAR, debug hooks).

Any sanitizer report aborts the run (halt_on_error=1) and fails the pytest invocation.
  python scripts/host_sanitize.py [--gpu]     -> writes a summary to stdout
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("GSB_SAN_DIR", "/tmp/gsb_san")
NVCC = "/usr/local/cuda/bin/nvcc"
SAN = "-fsanitize=address,undefined"


def sh(cmd, env=None, cwd=ROOT):
    print("+", " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=env, cwd=cwd, capture_output=True, text=True)


def runtime_libs():
    libs = []
    for name in ("libasan.so", "libubsan.so"):
        p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
        libs.append(p)
    return ":".join(libs)


def build_oracle():
    so = os.path.join(OUT, "liboracle_san.so")
    r = sh(["gcc", "-O1", "-g", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fno-omit-frame-pointer", SAN,
            "-fPIC", "-shared", "-pthread", "-o", so, os.path.join(ROOT, "oracle", "gsb_oracle.c"), "-lm"])
    if r.returncode:
        raise SystemExit(r.stderr)
    return so


def build_libgsb():
    so = os.path.join(OUT, "libgsb_san.so")
    from concurrent.futures import ThreadPoolExecutor

    def one(src):
        obj = os.path.join(OUT, os.path.basename(src)[:-3] + ".o")
        r = sh([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-g", "-lineinfo", "-std=c++17",
                "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xcompiler", "-fsanitize=address", "-Xcompiler",
                "-fsanitize=undefined", "-Xcompiler", "-fno-omit-frame-pointer", "-c", "-o", obj, src])
        if r.returncode:
            raise SystemExit(r.stderr)
        return obj

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(one, sorted(glob.glob(os.path.join(ROOT, "paper_2604_25459_b200", "csrc", "*.cu")))))
    r = sh([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", so, *objs, "-cudart", "shared",
            "-Xcompiler", "-fsanitize=address", "-Xcompiler", "-fsanitize=undefined",
            "-Xlinker", "-rpath=/usr/local/cuda/lib64"])
    if r.returncode:
        raise SystemExit(r.stderr)
    return so


def main():
    gpu = "--gpu" in sys.argv
    os.makedirs(OUT, exist_ok=True)
    env = dict(os.environ)
    env["LD_PRELOAD"] = runtime_libs()
    # CUDA maps memory where ASan's shadow gap sits; leaks of the interpreter are not ours
    env["ASAN_OPTIONS"] = "detect_leaks=0:halt_on_error=1:protect_shadow_gap=0:abort_on_error=0"
    env["UBSAN_OPTIONS"] = "halt_on_error=1:print_stacktrace=1"
    env["GSB_ORACLE_LIB"] = build_oracle()
    env["GSB_LIB_PATH"] = build_libgsb()
    results = {}
    oracle_tests = ["tests/test_oracle_pins.py", "tests/test_oracle_lidar.py", "tests/test_oracle_blur.py",
                    "tests/test_abi.py"]
    r = sh([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "not gpu", *oracle_tests],
           env=env)
    results["cpu: oracle pins + ABI validation"] = (r.returncode, r.stdout.strip().splitlines()[-1:] or [""])
    if r.returncode:
        print(r.stdout[-4000:], r.stderr[-4000:])
    if gpu:
        gpu_tests = ["tests/test_gpu_parity.py", "tests/test_gpu_static.py", "tests/test_gpu_lists.py",
                     "tests/test_gpu_lidar.py", "tests/test_gpu_obs.py", "tests/test_gpu_scores.py"]
        r = sh([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu and not slow",
                *gpu_tests], env=env)
        results["gpu: renders, static, lists, LiDAR, obs, scores through the sanitized host runtime"] = (
            r.returncode, r.stdout.strip().splitlines()[-1:] or [""])
        if r.returncode:
            print(r.stdout[-4000:], r.stderr[-4000:])
    print("host sanitizers (ASan + UBSan, halt_on_error=1):")
    ok = True
    for k, (rc, tail) in results.items():
        print(f"  {k}: {'clean' if rc == 0 else 'FAILED'} ({tail[0]})")
        ok &= rc == 0
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
