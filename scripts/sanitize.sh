export QC_JIT_CACHE=/tmp/qcjit_san
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 5 python scripts/run_circuit.py --circuit qft --n 14 --tile 10 --reps 2 --jit 0 > gpurun_out/san_${tool}_interp.txt 2>&1
  echo "$tool interp rc=$? $(grep -E 'ERROR SUMMARY|errors' gpurun_out/san_${tool}_interp.txt | tail -1)"
  timeout 600 compute-sanitizer --tool $tool --print-limit 5 python scripts/run_circuit.py --circuit tfxy --n 14 --steps 2 --tile 10 --reps 2 --jit 2 > gpurun_out/san_${tool}_jit.txt 2>&1
  echo "$tool jit rc=$? $(grep -E 'ERROR SUMMARY|errors' gpurun_out/san_${tool}_jit.txt | tail -1)"
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python scripts/run_circuit.py --circuit qft --n 14 --tile 10 --reps 2 --fusion 0 > gpurun_out/san_memcheck_unfused.txt 2>&1
echo "memcheck unfused rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/san_memcheck_unfused.txt | tail -1)"
