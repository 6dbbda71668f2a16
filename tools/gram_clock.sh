python tools/gram_clock.py 0 4 5 6
cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 umma_rate.cu -o /tmp/umma_rate && /tmp/umma_rate
