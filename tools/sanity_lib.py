"""Launch one-kernel libraries through ctypes after torch initialised CUDA, built like
liboaa.so (run under compute-sanitizer; see profiles/r02_sanitizer_*.txt):
  one .cu compiled straight to a .so, and two objects (nvcc -c) linked with -lcudart."""
import ctypes, os, subprocess, sys
import torch
here = os.path.dirname(os.path.abspath(__file__))
mb = os.path.join(here, "microbench")
arch = ["-gencode", "arch=compute_100a,code=sm_100a"]
subprocess.run(["nvcc"] + arch + ["-shared", "-Xcompiler", "-fPIC", os.path.join(mb, "sanity_lib.cu"), "-o",
                "/tmp/libsanity.so"], check=True)
for f in ["sanity_lib", "sanity_lib2"]:
    subprocess.run(["nvcc"] + arch + ["-O3", "-Xcompiler", "-fPIC", "-c", os.path.join(mb, f + ".cu"), "-o",
                    f"/tmp/{f}.o"], check=True)
subprocess.run(["nvcc"] + arch + ["-shared", "-o", "/tmp/libsanity2.so", "/tmp/sanity_lib.o", "/tmp/sanity_lib2.o",
                "-lcudart"], check=True)
x = torch.zeros(32, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
which = sys.argv[1] if len(sys.argv) > 1 else "one"
if which == "one":
    lib = ctypes.CDLL("/tmp/libsanity.so")
    rc = lib.sanity_launch(ctypes.c_void_p(x.data_ptr()), s)
else:
    lib = ctypes.CDLL("/tmp/libsanity2.so")
    rc = lib.sanity_launch2(ctypes.c_void_p(x.data_ptr()), s) or lib.sanity_launch(ctypes.c_void_p(x.data_ptr()), s)
torch.cuda.synchronize()
print(which, "rc", rc, "sum", float(x.sum()))
