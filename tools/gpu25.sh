mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded" -m "gpu" 2>&1 | tail -3
timeout 300 python tools/time_ops.py 256,96,256,27,5
timeout 300 python tools/time_ops.py 128,64,128,224,8
timeout 300 python tools/time_ops.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_alex5.csv python tools/time_ops.py 256,96,256,27,5 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_shard5.csv python tools/time_ops.py 128,64,128,224,8 > /dev/null 2>&1
