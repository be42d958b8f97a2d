python scripts/trace_gemm.py 16 28672 4096 2>&1
python scripts/trace_gemm.py 16 4096 4096 2>&1
python scripts/trace_gemm.py 16 28672 4096 16 1 2>&1
