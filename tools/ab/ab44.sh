# ragged: all e^{-x} of a lane's elements before the queue decisions (libboys.so) vs HEAD (libboys_prev.so)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -k "ragged or smoke" 2>&1 | tail -1
bash tools/ab/ab22.sh
