# experiment builds on the GPU box: tools/exp_build.sh "-DFLAG ..." rebuilds libhmxg.so in place
set -e
cd "$(dirname "$0")/../paper_1812_07152_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -shared $1 -o ../libhmxg.so hmxg.cu krows.cu compress.cu plan.cpp cdsfile.cpp
