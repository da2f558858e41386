for L in _mb/libS.so _mb/libT.so _mb/libU.so _mb/libV.so; do
  SP_LIBRARY=$PWD/$L timeout 300 python -m pytest tests/test_lookup_gpu.py -q -x -k "forward or golden or generator" > gpurun_out/ab_test_$(basename $L).log 2>&1; echo "$L rc=$?" >> gpurun_out/ab4.log
  SP_LIBRARY=$PWD/$L timeout 200 python tools/sort_probe.py cfg3 20 >> gpurun_out/ab4.log 2>&1
  SP_LIBRARY=$PWD/$L timeout 200 python tools/sort_probe.py cfg3 20 >> gpurun_out/ab4.log 2>&1
done
