timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for s in 5 6 7 5; do echo "SBL=$s"; OAA_SBL=$s timeout 120 python tools/time_ops.py 256,96,256,27,5; OAA_SBL=$s timeout 300 python tools/time_ops.py 128,64,128,224,8; done
