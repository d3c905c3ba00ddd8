mkdir -p gpurun_out/g100
OAA_TC_BSPLIT=1 timeout 600 ncu --set full --clock-control none -k regex:oaa_bin_gemm -s 1 -c 1 -o gpurun_out/g100/new python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
OAA_LIB=$PWD/tmp_oldlib/liboaa.so timeout 600 ncu --set full --clock-control none -k regex:oaa_bin_gemm -s 1 -c 1 -o gpurun_out/g100/old python tools/prof_step.py 2 fwd 256,96,256,27,5 > /dev/null 2>&1
