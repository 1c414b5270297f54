# Round-2 final evidence (latest code): GPU tests, smoke, bench lines of every config + the
# reference arm, the C2 phase trace, launch lists, ncu captures of the hot kernels.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 400 gpurun_out/bench_c2.json
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 200 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 300 gpurun_out/bench_$c.json; done
timeout 600 python bench.py --config c5 --sharded --steps 50 --warmup 3 > gpurun_out/bench_c5_sharded.json 2> gpurun_out/bench_c5_sharded.err
timeout 600 python bench.py --config c5 --sharded --exchange device --steps 50 --warmup 3 > gpurun_out/bench_c5_sharded_devx.json 2> gpurun_out/bench_c5_sharded_devx.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; tail -c 300 gpurun_out/bench_reference.json
FIER_LIB=paper_2508_08256_b200/libfier_cuda_trace.so timeout 300 python tools/step_trace.py --config c2 --reps 12 > gpurun_out/step_trace_c2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_fused -s 6 -c 1 -o gpurun_out/r2_c2_step_fused python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_mma -s 2 -c 1 -o gpurun_out/r2_c4_score_mma python tools/kbench.py --config c4 --reps 3 --layers 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tr_row -s 1 -c 1 -o gpurun_out/r2_c4_tr_row python tools/kbench.py --config c4 --reps 3 --layers 2 > /dev/null 2>&1
ls -la gpurun_out
