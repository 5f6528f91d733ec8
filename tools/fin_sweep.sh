for t in base "$@"; do
  if [ "$t" = base ]; then L=paper_2508_16508_b200/libabmx_cuda.so; else L=build/variants/$t/libabmx_cuda.so; fi
  echo "== $t"
  ABMX_CUDA_LIB=$L timeout 200 python tools/prof_finance.py 2>&1 | tail -1
  ABMX_CUDA_LIB=$L timeout 300 python -m pytest -q -x tests/test_finance_gpu.py 2>&1 | tail -1
done
