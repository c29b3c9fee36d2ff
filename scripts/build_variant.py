"""Build libtm_<name>.so with extra nvcc -D flags for same-box A/B runs
(TM_LIB_VARIANT=<name>).  usage: python scripts/build_variant.py name -DFOO=1 ..."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1509_04863_b200._build import FLAGS, NVCC, CSRC  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
objs, procs = [], []
os.makedirs("/tmp/tm_variant", exist_ok=True)
for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
    obj = f"/tmp/tm_variant/{name}_{os.path.basename(src)}.o"
    procs.append(subprocess.Popen([NVCC, *FLAGS, *extra, "-c", src, "-o", obj]))
    objs.append(obj)
assert all(p.wait() == 0 for p in procs)
out = os.path.join(ROOT, "paper_1509_04863_b200", f"libtm_{name}.so")
subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out, *objs])
print(out)
