# A/B/n: bench.py with the working-tree lib and tools/var/libfier_<v>.so for each v, alternated 3x.
# usage: bash tools/gpu_abn.sh CONFIG "v1 v2 ..." [extra bench args]
cfg=$1; vs=$2; shift 2
for i in 1 2 3; do
  for v in new $vs; do
    if [ $v = new ]; then L=""; else L=tools/var/libfier_$v.so; fi
    FIER_LIB=$L timeout 300 python bench.py --config $cfg --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print('$v', '$cfg', d['value'], d['e2e']['value'], d.get('per_kernel_us'))
" | tee -a gpurun_out/abn_$cfg.txt
  done
done
