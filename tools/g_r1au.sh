mkdir -p gpurun_out
for v in main b8 main b8; do
  if [ $v = main ]; then L=""; else L="libvoxmap_b200_$v.so"; fi
  VOXMAP_B200_LIB=$L timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/au_$v.txt 2>&1
  echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/au_$v.txt | head -1) $(grep -o '"fold_ms": [0-9.]*' gpurun_out/au_$v.txt)" >> gpurun_out/au_summary.txt
done
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/au_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/au_pytest.txt
