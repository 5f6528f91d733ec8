for r in 1 2; do
for v in base st4 st6 cc2 cc4; do
  if [ $v = base ]; then L=paper_2508_16508_b200/libabmx_cuda.so; else L=build/variants/$v/libabmx_cuda.so; fi
  ABMX_CUDA_LIB=$L python bench.py --no-ensemble --no-traffic --no-finance --no-agents --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['kernel_table']['entries']; print('$v', {k: round(v['us'],1) for k,v in e.items()})"
done; done
