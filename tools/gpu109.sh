for r in 3 6; do echo ring=$r; OAA_LIB=$PWD/exp_r$r/liboaa.so timeout 120 python tools/time_ops.py; done
echo ring=4; timeout 120 python tools/time_ops.py
