# step_trace of the baseline trace build and every tools/var/*_trace.so variant
for lib in paper_2508_08256_b200/libfier_cuda_trace.so tools/var/*_trace.so; do
  echo "=== $lib"
  FIER_LIB=$lib timeout 300 python tools/step_trace.py --config ${CFG:-c2} --reps ${REPS:-12} 2>&1 | grep -v "^max active" | head -${LINES_:-40}
done
