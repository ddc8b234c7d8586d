# compute-sanitizer over the interpreting (AOT) and NVRTC-specialised fused passes, and the per-gate kernels
export QC_JIT_CACHE=/tmp/qcjit_san
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 5 python scripts/run_circuit.py --circuit qft --n 14 --tile 10 --reps 2 --jit 0 > gpurun_out/san_${tool}_interp.txt 2>&1
  echo "$tool interp rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_interp.txt | tail -1)"
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python scripts/run_circuit.py --circuit tfxy --n 16 --steps 3 --reps 2 --jit 2 > gpurun_out/san_${tool}_jit.txt 2>&1
  echo "$tool jit (TFXY-16, remap, 16-warp passes) rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_jit.txt | tail -1)"
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python scripts/run_circuit.py --circuit qft --n 15 --prec c64 --reps 2 --jit 2 > gpurun_out/san_${tool}_jit64.txt 2>&1
  echo "$tool jit (QFT-15 c64) rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_jit64.txt | tail -1)"
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python scripts/run_circuit.py --circuit qft --n 14 --tile 10 --reps 2 --fusion 0 > gpurun_out/san_memcheck_unfused.txt 2>&1
echo "memcheck unfused rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/san_memcheck_unfused.txt | tail -1)"
