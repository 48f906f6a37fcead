# ragged A/B: old library (ab_libs/libboys_old.so) vs the current build; ragged parity tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_boundary.py -q -m gpu -x -k "ragged or Ragged" > gpurun_out/pytest_v.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_v.log; tail -n 3 gpurun_out/pytest_v.log
for i in 1 2; do
for lib in $EXTRA_LIBS ab_libs/libboys_old.so paper_2504_07637_b200/libboys.so; do
echo $lib; BOYS_LIB=$PWD/$lib timeout 300 python tools/ragged_rate.py
done
done
