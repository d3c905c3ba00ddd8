timeout 900 python -m pytest tests -x -q -m gpu -k "tensor_core_path or alexnet or sharded or bin_gemm" 2>&1 | tail -3
