# k_accept CTA size for the C4 long road: the default build vs build/variants/na*
for t in base "$@"; do
  if [ "$t" = base ]; then L=paper_2508_16508_b200/libabmx_cuda.so; else L=build/variants/$t/libabmx_cuda.so; fi
  echo "== $t"
  ABMX_CUDA_LIB=$L timeout 200 python tools/prof_traffic.py 2>&1 | head -2
done
