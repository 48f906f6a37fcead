# same-box A/B: compacted e^{-x} in ragged chunks (libboys.so) vs every-lane e^{-x} (libboys_prev.so)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -k "ragged or smoke" > gpurun_out/pytest_ragged.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ragged.log
tail -2 gpurun_out/pytest_ragged.log
bash tools/ab/ab22.sh
