for v in "" _build_oaa_exp_no_wait/liboaa.so _build_oaa_exp_relaxed_publish/liboaa.so _build_oaa_exp_no_wait_oaa_exp_relaxed_publish/liboaa.so; do
  if [ -n "$v" ]; then export OAA_LIB=$PWD/paper_1601_06815_b200/$v; else unset OAA_LIB; fi
  timeout 300 python tools/time_ops.py
done
