#!/bin/bash
# usage: mkvar.sh name "-DFOO=1 ..."   -> _exp/name/{paper_1209_6449_b200,synth,tools}
set -e
cd /root/repo
d=_exp/$1; rm -rf $d; mkdir -p $d
cp -r paper_1209_6449_b200 synth tools $d/
rm -f $d/paper_1209_6449_b200/libepsm.so
NCCL=$(python -c "import sys; sys.path.insert(0,'paper_1209_6449_b200'); import build; print(build.nccl_include())")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC -Xcompiler -fvisibility=default $2 -I include -I paper_1209_6449_b200/csrc -I $NCCL -o $d/paper_1209_6449_b200/libepsm.so paper_1209_6449_b200/csrc/epsm.cu paper_1209_6449_b200/csrc/epsm_sharded.cu paper_1209_6449_b200/csrc/epsm_multi.cu paper_1209_6449_b200/csrc/epsm_host.cu paper_1209_6449_b200/csrc/epsm_long.cu -ldl
touch $d/paper_1209_6449_b200/libepsm.so
