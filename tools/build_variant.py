"""Builds a variant of the engine library with extra nvcc defines, for A/B
probes on the box (not the product build):

    python tools/build_variant.py /tmp/out.so -DCCLP_STREAM_HINT=1
    CCLP_CU_LIB=/tmp/out.so python tools/probe_ab.py ...
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_24429_b200 import build as b  # noqa: E402

out, defs = os.path.abspath(sys.argv[1]), sys.argv[2:]
objdir = out + ".obj"
os.makedirs(objdir, exist_ok=True)


def one(src):
    obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
    subprocess.run([b.nvcc(), *b.NVCC_FLAGS, *defs, "-c", "-o", obj, os.path.join(b.HERE, src)],
                   check=True, cwd=b.HERE)
    return obj


with ThreadPoolExecutor(len(b.SOURCES)) as ex:
    objs = list(ex.map(one, b.SOURCES))
subprocess.run([b.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs],
               check=True)
print(out)
