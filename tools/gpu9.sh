for v in "" "_build_oaa_ring_depth=4_oaa_publish_every=2/liboaa.so" "_build_oaa_engine_minb=2_oaa_ring_depth=4_oaa_publish_every=2/liboaa.so"; do
  if [ -n "$v" ]; then export OAA_LIB=$PWD/paper_1601_06815_b200/$v; else unset OAA_LIB; fi
  timeout 300 python tools/time_ops.py
done
export OAA_LIB="$PWD/paper_1601_06815_b200/_build_oaa_engine_minb=2_oaa_ring_depth=4_oaa_publish_every=2/liboaa.so"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small_grid and (8 or 5)" 2>&1 | tail -2
