"""Build experimental liblfem.so variants (compile-time tile-kernel knobs) under scripts/variants/<name>/.
usage: build_variants.py name=-DFLAG=V,-DFLAG2=V ..."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14035_b200 import build as b
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants")
jobs = []
for spec in sys.argv[1:]:
    name, flags = spec.split("=", 1)
    od = os.path.join(out, name); os.makedirs(od, exist_ok=True)
    objs = []
    for src in b.sources():
        obj = os.path.join(od, os.path.basename(src) + ".o")
        jobs.append(subprocess.Popen([b.NVCC, *b.NVCC_FLAGS, *flags.split(","), "-c", src, "-o", obj])); objs.append(obj)
    jobs.append((od, objs))
for j in jobs:
    if isinstance(j, subprocess.Popen): j.wait()
for j in jobs:
    if isinstance(j, tuple):
        od, objs = j
        subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", os.path.join(od, "liblfem.so"), *objs], check=True)
        print(od, "ok")
