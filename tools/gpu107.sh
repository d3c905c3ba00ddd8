for s in 3 4 5 3 4 5; do echo "SBL=$s"; OAA_SBL=$s timeout 120 python tools/time_ops.py 256,96,256,27,5; done
for s in 3 5; do echo "SBL=$s"; OAA_SBL=$s timeout 300 python tools/time_ops.py 128,64,128,224,8; done
