for mb in 20 30 40 60 200; do echo "band=$mb"; CT_GEMM_BAND_MB=$mb timeout 200 python tools/gemm_swiglu_bench.py 2>&1 | tail -4 | python -c "
import sys,json
for l in sys.stdin:
  j=json.loads(l); print(j['rows'], j['fused_us'], j['fused_tflops'], j['cublas_mm_tflops'])"; done
