mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck python tools/sanitize_run.py > gpurun_out/san_memcheck.txt 2>&1
timeout 1200 $CS --tool racecheck python tools/racecheck_run.py > gpurun_out/san_racecheck.txt 2>&1
timeout 1200 $CS --tool synccheck python tools/racecheck_run.py > gpurun_out/san_synccheck.txt 2>&1
timeout 1200 $CS --tool initcheck python tools/racecheck_run.py > gpurun_out/san_initcheck.txt 2>&1
for f in gpurun_out/san_*.txt; do echo "== $f"; tail -4 $f; done
timeout 300 python tools/prof_pop.py fp64 > gpurun_out/san_timing.txt 2>&1; cat gpurun_out/san_timing.txt
timeout 900 python -m pytest tests/test_gpu_full_length.py tests/test_gpu_parity.py tests/test_cv.py -m gpu -q -x 2>&1 | tail -2
