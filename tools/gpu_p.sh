bash tools/gpu_abn.sh c2 "l2 l6 nst3"
