mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core or tcgen05" 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "alexnet or sharded" -m "gpu" 2>&1 | tail -15
timeout 300 python tools/time_ops.py 256,96,256,27,5
timeout 300 python tools/time_ops.py 128,64,128,224,8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_alex3.csv python tools/time_ops.py 256,96,256,27,5 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_shard3.csv python tools/time_ops.py 128,64,128,224,8 > /dev/null 2>&1
