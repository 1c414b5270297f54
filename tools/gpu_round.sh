set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
for c in c2 c1 c3 c4; do timeout 600 python bench.py --config $c --steps 400 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 3000 gpurun_out/bench_$c.json; done
timeout 300 python tools/kbench.py --config c2 > gpurun_out/kbench_c2.txt 2>&1; cat gpurun_out/kbench_c2.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/launches.py gpurun_out/launches_c2.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score128|attn_tc|topk_kernel|append' -s 20 -c 8 -o gpurun_out/prof_c2 python tools/kbench.py --config c2 --reps 5 --layers 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
