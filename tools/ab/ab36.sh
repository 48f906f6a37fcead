# A/B: ragged recursion steps with one merged predicate per element (libboys.so) vs libboys_prev.so
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -k "ragged or smoke or graph" > gpurun_out/pytest_ragged.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ragged.log
tail -2 gpurun_out/pytest_ragged.log
bash tools/ab/ab22.sh
