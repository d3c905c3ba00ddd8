timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for b in 0 1; do echo "BSPLIT=$b"; OAA_TC_BSPLIT=$b timeout 120 python tools/time_ops.py 256,96,256,27,5; OAA_TC_BSPLIT=$b timeout 300 python tools/time_ops.py 128,64,128,224,8; done
echo default; timeout 120 python tools/time_ops.py 256,96,256,27,5
