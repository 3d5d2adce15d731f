# diagnostic engine builds (not shipped): libamvm_<tag>.so = amvm.cu with extra -D flags + the shipped other units
set -e
cd "$(dirname "$0")/../paper_2508_13437_b200"
tag=$1; shift
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I ../include"
/usr/local/cuda/bin/nvcc $F "$@" -c -o _obj/amvm_$tag.o csrc/amvm.cu
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libamvm_$tag.so _obj/amvm_$tag.o _obj/amvm_aux.o _obj/amvm_score.o
echo built libamvm_$tag.so
