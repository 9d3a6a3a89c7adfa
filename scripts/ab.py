"""A/B timing of builds of libgsb in one GPU session (interleaved bench runs).

  here:    python scripts/ab.py build <git-ref-A>      # A = csrc at that ref, B = working tree
           python scripts/ab.py variants N1="-DX=1" N2="-DX=2 -DY=3" ...   # working tree + macros
  on GPU:  python scripts/ab.py run [reps] [bench args...]   # every ab/libgsb_*.so, interleaved
Writes ab/libgsb_<name>.so (in-tree, so they travel with gpurun).
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "ab")


def build(ref):
    from paper_2604_25459_b200 import build as b
    os.makedirs(OUT, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.check_call(f"git -C {ROOT} archive {ref} paper_2604_25459_b200/csrc include | tar -x -C {tmp}",
                              shell=True)
        srcs = sorted(os.path.join(tmp, "paper_2604_25459_b200", "csrc", f)
                      for f in os.listdir(os.path.join(tmp, "paper_2604_25459_b200", "csrc")) if f.endswith(".cu"))
        subprocess.check_call([b.NVCC, *b.ARCH, *b.FLAGS, "-shared", "-o", os.path.join(OUT, "libgsb_A.so"), *srcs,
                               *b.LINK])
    subprocess.check_call([b.NVCC, *b.ARCH, *b.FLAGS, "-shared", "-o", os.path.join(OUT, "libgsb_B.so"),
                           *b.sources(), *b.LINK])


def variants(specs):
    from concurrent.futures import ThreadPoolExecutor
    from paper_2604_25459_b200 import build as b
    os.makedirs(OUT, exist_ok=True)
    for f in os.listdir(OUT):
        if f.startswith("libgsb_"):
            os.remove(os.path.join(OUT, f))

    def one(spec):
        name, _, defs = spec.partition("=")
        subprocess.check_call([b.NVCC, *b.ARCH, *b.FLAGS, *defs.split(), "-shared", "-o",
                               os.path.join(OUT, f"libgsb_{name}.so"), *b.sources(), *b.LINK])

    with ThreadPoolExecutor(len(specs)) as ex:
        list(ex.map(one, specs))


def run(reps, args):
    names = sorted(f[len("libgsb_"):-3] for f in os.listdir(OUT) if f.startswith("libgsb_") and f.endswith(".so"))
    res = {v: [] for v in names}
    for r in range(reps):
        for v in names:
            env = dict(os.environ, GSB_LIB_PATH=os.path.join(OUT, f"libgsb_{v}.so"))
            out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-e2e", "--no-cpu-baseline",
                                  *args], capture_output=True, text=True, env=env, cwd=ROOT)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            if not line:
                print(v, "failed", out.stderr[-2000:])
                continue
            d = json.loads(line[-1])
            st = d.get("stage_ms_per_step", {})
            res[v].append((d["value"], st.get("composite_ms"), st.get("project_ms"), st.get("emit_ms")))
            print(v, r, json.dumps(res[v][-1]), flush=True)
    for v in names:
        if not res[v]:
            continue
        vals = sorted(x[0] for x in res[v])
        comp = sorted(x[1] for x in res[v])
        print(v, "median value", vals[len(vals) // 2], "median composite_ms", comp[len(comp) // 2])


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2])
    elif sys.argv[1] == "variants":
        variants(sys.argv[2:])
    else:
        reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
        run(reps, sys.argv[3:])
