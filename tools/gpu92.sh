timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 120 python tools/time_ops.py 256,96,256,27,5
timeout 300 python tools/time_ops.py 128,64,128,224,8
echo NOHI
OAA_TC_NOHI=1 timeout 900 python -m pytest tests -x -q -m gpu -k "tc or alex or sharded or filter or engine" 2>&1 | tail -2
OAA_TC_NOHI=1 timeout 120 python tools/time_ops.py 256,96,256,27,5
OAA_TC_NOHI=1 timeout 300 python tools/time_ops.py 128,64,128,224,8
