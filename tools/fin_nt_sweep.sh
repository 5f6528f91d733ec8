# finance small-window CTA size: the default build vs build/variants/fsn*
for t in base "$@"; do
  if [ "$t" = base ]; then L=paper_2508_16508_b200/libabmx_cuda.so; else L=build/variants/$t/libabmx_cuda.so; fi
  echo "== $t"; ABMX_CUDA_LIB=$L python tools/fin_one_market.py
done
