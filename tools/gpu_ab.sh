# A/B timing of library variants: usage gpu_ab.sh "<tool.py args>" lib1 lib2 ... (two alternating passes)
mkdir -p gpurun_out
tool=$1; shift
for i in 1 2; do
for lib in "$@"; do
echo $lib; BOYS_LIB=$PWD/$lib timeout 300 python $tool
done
done
