"""Build experimental liblfem.so variants (tile configs) under scripts/variants/."""
import os, subprocess, sys, glob
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14035_b200 import build as b
VARS = {"t192m2r256": (192, 2, 256), "t128m3r160": (128, 3, 160), "t256m1r384": (256, 1, 384), "t384m1r512": (384, 1, 512)}
names = sys.argv[1:] or list(VARS)
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants")
procs = []
for n in names:
    th, mb, r = VARS[n]
    od = os.path.join(out, n); os.makedirs(od, exist_ok=True)
    objs = []
    for src in b.sources():
        obj = os.path.join(od, os.path.basename(src) + ".o")
        cmd = [b.NVCC, *b.NVCC_FLAGS, f"-DLFEM_P2T_THREADS={th}", f"-DLFEM_P2T_MINB={mb}", f"-DLFEM_P2T_R={r}", "-c", src, "-o", obj]
        procs.append(subprocess.Popen(cmd)); objs.append(obj)
    for p in procs: p.wait()
    procs = []
    subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", os.path.join(od, "liblfem.so"), *objs], check=True)
    print(n, "ok")
