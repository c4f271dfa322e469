# Scratch: short-k GEMMs (fp32 C) on the 256 x 256 plan with more staging tiles in flight (libs built with
# TLB_NVCC_EXTRA="-DTLB_UMMA_STAGES=4 -DTLB_UMMA_EPIBUFS=3")
for lib in "" tools/probes/libtlb_s4e2.so tools/probes/libtlb_s4e3.so; do
  echo "=== lib ${lib:-default (6 stages, 1 staging tile per half)}"
  for shape in "8192 8192 1024" "4096 4096 1024" "4096 4096 2048" "8192 8192 2048" "32768 1024 1152"; do
    TLB_LIB=$lib TLB_GEMM_WIDE=0 python tools/gemm_probe.py $shape 30 | tail -1
  done
  TLB_LIB=$lib TLB_GEMM_WIDE=0 TLB_GEMM_DEBUG=1 python tools/gemm_probe.py 8192 8192 1024 30 | tail -1
done
