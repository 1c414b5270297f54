set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c1 --steps 200 --warmup 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
FIER_LIB=paper_2508_08256_b200/libfier_cuda_trace.so timeout 300 python tools/step_trace.py --config c2 --reps 12 > gpurun_out/step_trace_c2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_fused -s 6 -c 1 -o gpurun_out/r2_c2_step_fused python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
