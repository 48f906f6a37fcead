mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_m.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_m.log; tail -n 2 gpurun_out/pytest_m.log
for i in 1 2; do
for L in old A both; do BOYS_LIB=$PWD/ab_libs/libboys_$L.so timeout 300 python tools/dense_rate.py; done
timeout 300 python tools/dense_rate.py
for L in old A both; do BOYS_LIB=$PWD/ab_libs/libboys_$L.so timeout 200 python tools/cfg1_stream.py; done
timeout 200 python tools/cfg1_stream.py
for L in old both; do BOYS_LIB=$PWD/ab_libs/libboys_$L.so timeout 200 python tools/ragged_rate.py; done
timeout 200 python tools/ragged_rate.py
done
