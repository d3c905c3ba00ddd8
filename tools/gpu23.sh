mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core or tcgen05" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "alexnet or sharded" -m "gpu" 2>&1 | tail -3
timeout 300 python tools/time_ops.py 256,96,256,27,5
timeout 300 python tools/time_ops.py 128,64,128,224,8
