"""Experiment builds: recompile some sources with extra nvcc flags and link them with the other objects of
build/ into paper_2410_16135_b200/libvnm_<name>.so (loaded when VNM_LIB points at it; never the product).
Usage: python scripts/build_variant.py NAME "FLAGS" file.cu [file.cu ...]"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16135_b200 import build as B

name, flags, files = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
B.build()
srcdir, all_files = B.LIBS[os.path.join(B.HERE, "libvnm.so")]
vdir = os.path.join(B.HERE, "build_var_" + name)
os.makedirs(vdir, exist_ok=True)
objs = []
for f in all_files:
    if f in files:
        o = os.path.join(vdir, f + ".o")
        subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, *flags, "-I", B.CSRC, "-c", "-o", o, os.path.join(srcdir, f)])
        objs.append(o)
    else:
        objs.append(os.path.join(B.HERE, "build", f + ".o"))
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(B.HERE, f"libvnm_{name}.so"), *objs, "-lcudart"])
print("built", f"libvnm_{name}.so")
