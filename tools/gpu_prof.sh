# per-kernel ncu --set full captures of the C2 decode step kernels (one launch each)
set -x
./tools/mma_probe > gpurun_out/mma_probe.txt 2>&1; cat gpurun_out/mma_probe.txt
for k in score128 topk_kernel attn_tc_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o gpurun_out/prof_c2_$k python tools/kbench.py --config c2 --reps 3 --layers 2 > gpurun_out/ncu_$k.log 2>&1
  tail -2 gpurun_out/ncu_$k.log
done
