# Round state check: GPU tests, smoke, bench lines of every config, C2 phase trace.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 1500 gpurun_out/bench_$c.json; done
FIER_LIB=paper_2508_08256_b200/libfier_cuda_trace.so timeout 300 python tools/step_trace.py --config c2 --reps 12 > gpurun_out/step_trace_c2.txt 2>&1; tail -30 gpurun_out/step_trace_c2.txt
