nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier_bench scripts/barrier_bench.cu && /tmp/barrier_bench
