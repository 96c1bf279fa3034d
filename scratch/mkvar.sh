#!/bin/bash
# scratch/mkvar.sh NAME "-DFLAG ..." : library variant with unet_cluster.cu compiled with extra flags,
# in scratch/var_NAME (a copy of the package; run scratch/step_time.py from there)
set -e
N=$1; F=$2
D=scratch/var_$N
rm -rf $D; mkdir -p $D/scratch
cp -r paper_2509_09560_b200 $D/; rm -rf $D/paper_2509_09560_b200/csrc/build
cp scratch/step_time.py $D/scratch/
cd paper_2509_09560_b200/csrc
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr --extended-lambda $F -c unet_cluster.cu -o /tmp/uc_$N.o
OBJS=$(ls build/*.o | grep -v unet_cluster)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../$D/paper_2509_09560_b200/libauras_b200.so $OBJS /tmp/uc_$N.o -lcudart
