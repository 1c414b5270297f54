timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_shard.py -x -q 2>&1 | tail -3
for c in c2 c3 c4; do timeout 300 python tools/kbench.py --config $c 2>&1 | grep -E "topk|score"; done
for cl in 2 4; do echo cluster $cl; FIER_TOPK_CLUSTER=$cl timeout 300 python tools/kbench.py --config c2 2>&1 | grep topk; done
