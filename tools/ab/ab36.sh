# A/B: ragged (libboys.so) vs libboys_prev.so (ab36: merged step predicate; ab37: unpredicated full-chunk loads)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -k "ragged or smoke or graph" > gpurun_out/pytest_ragged.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ragged.log
tail -2 gpurun_out/pytest_ragged.log
bash tools/ab/ab22.sh
