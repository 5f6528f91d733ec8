for L in build/variants/trfbase/libabmx_cuda.so paper_2508_16508_b200/libabmx_cuda.so; do
  echo "== $L"
  for i in 1 2 3; do ABMX_CUDA_LIB=$L python tools/prof_traffic_ens.py 1000; done
done
python -m pytest -q -x tests/test_traffic_gpu.py
