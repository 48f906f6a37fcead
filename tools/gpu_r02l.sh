mkdir -p gpurun_out
for i in 1 2; do
BOYS_LIB=$PWD/ab_libs/libboys_old.so timeout 300 python tools/dense_rate.py
timeout 300 python tools/dense_rate.py
BOYS_LIB=$PWD/ab_libs/libboys_old.so SINGLE_OUT=1 timeout 300 python tools/dense_rate.py
SINGLE_OUT=1 timeout 300 python tools/dense_rate.py
done
