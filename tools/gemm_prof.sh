GDP_NVCC_EXTRA=-DGEMM_PROF python tools/gemm_prof.py 2>&1 | grep GPROF | tail -16
