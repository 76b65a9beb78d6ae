"""Build a variant of libgivens.so with extra nvcc defines into exp/lib_<name>.so (A/B timing with
tools/ab_libs.sh). usage: python tools/variant.py NAME [-DFOO=1 ...] [--rings W_L,W_L,...]
Only the listed ring objects are rebuilt with the defines (default: all); the rest are reused
from paper_2106_00003_b200/build_obj."""
import os, subprocess, sys, shutil
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2106_00003_b200 import build as b

name, defs, rings = sys.argv[1], [], None
for a in sys.argv[2:]:
    if a.startswith("--rings="):
        rings = [tuple(int(x) for x in r.split("_")) for r in a.split("=", 1)[1].split(",")]
    else:
        defs.append(a)
out = os.path.join(ROOT, "exp", "obj_" + name)
os.makedirs(out, exist_ok=True)
jobs, objs = [], []
go = os.path.join(out, "givens.o")
jobs.append([b.NVCC, *b.FLAGS, *defs, "-c", "-o", go, b.SRC]); objs.append(go)
for w, l in b.RING_CONFIGS:
    if rings is None or (w, l) in rings:
        o = os.path.join(out, f"ring_{w}_{l}.o")
        jobs.append([b.NVCC, *b.FLAGS, *defs, f"-DRING_W={w}", f"-DRING_L={l}", "-c", "-o", o, b.RING_SRC])
    else:
        o = os.path.join(b.OBJ, f"ring_{w}_{l}.o")
    objs.append(o)
with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
    list(ex.map(subprocess.check_call, jobs))
lib = os.path.join(ROOT, "exp", f"lib_{name}.so")
subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs])
print(lib)
