for i in 1 2; do for L in old minb2 epl3 minb4; do BOYS_LIB=$PWD/ab_libs/libboys_$L.so timeout 200 python tools/ragged_rate.py cfg4f32; done; done
