"""Launch the one-kernel library tools/microbench/sanity_lib.cu through ctypes after torch
initialised CUDA (run under compute-sanitizer; see profiles/r02_sanitizer_*.txt)."""
import ctypes, os, subprocess, sys
import torch
here = os.path.dirname(os.path.abspath(__file__))
so = "/tmp/libsanity.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                os.path.join(here, "microbench", "sanity_lib.cu"), "-o", so], check=True)
lib = ctypes.CDLL(so)
x = torch.zeros(32, device="cuda")
rc = lib.sanity_launch(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("rc", rc, "sum", float(x.sum()))
