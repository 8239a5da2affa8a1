nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rowbw scripts/rowbw_bench.cu && /tmp/rowbw
