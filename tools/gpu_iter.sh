timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -k "score or decode_step or c2_shape or fused" 2>&1 | tail -5
timeout 300 python tools/kbench.py --config c2 2>&1 | grep score
timeout 300 python tools/kbench.py --config c3 2>&1 | grep score
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_mma -s 4 -c 1 -o gpurun_out/prof_score_mma_c2 python tools/kbench.py --config c2 --reps 3 --layers 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_mma -s 4 -c 1 -o gpurun_out/prof_score_mma_c3 python tools/kbench.py --config c3 --reps 3 --layers 2 > /dev/null 2>&1
ls gpurun_out
