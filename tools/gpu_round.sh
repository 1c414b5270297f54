# Round measurement: GPU tests, smoke, bench lines for every config, launch list and
# ncu captures of the decode step (copied into profiles/ afterwards).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 200 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 3000 gpurun_out/bench_$c.json; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; tail -c 1500 gpurun_out/bench_reference.json
FIER_LIB=paper_2508_08256_b200/libfier_cuda_trace.so timeout 300 python tools/step_trace.py --config c2 --reps 12 > gpurun_out/step_trace_c2.txt 2>&1; cat gpurun_out/step_trace_c2.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_fused -s 6 -c 1 -o gpurun_out/prof_c2_step_fused python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:attn_tc_kernel.*false" -s 2 -c 1 -o gpurun_out/prof_c2_full_kv python tools/kbench.py --config c2 --reps 3 --layers 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_mma -s 8 -c 1 -o gpurun_out/prof_c3_score_mma python tools/kbench.py --config c3 --reps 3 --layers 2 > /dev/null 2>&1
ls gpurun_out
