timeout 600 ncu --set full --clock-control none -k regex:gather_cpasync -s 3 -c 1 -o gpurun_out/prof_gprobe ./tools/gather_probe > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ws -s 4 -c 1 -o gpurun_out/prof_ws_c2 python tools/kbench.py --config c2 --reps 3 --layers 2 > /dev/null 2>&1
