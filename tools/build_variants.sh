#!/bin/bash
# Build library variants in parallel:
#   build_variants.sh name1 "-DX=1" name2 "-DY=0@/path/to/rq_kernels.cu" ...
# flags may carry "@file" = an alternative rq_kernels.cu for that variant.
# -> paper_1408_5526_b200/librqmc_b200_<name>.so (for RQMC_B200_LIB A/B runs)
R=/root/repo
while [ $# -ge 2 ]; do
  n=$1; f=${2%%@*}; alt=""; [[ "$2" == *@* ]] && alt=${2#*@}; shift 2
  ( d=$(mktemp -d); mkdir -p $d/include $d/pkg/csrc
    cp $R/include/*.h $d/include/; cp $R/paper_1408_5526_b200/csrc/{*.cu,*.cuh,*.h,*.inc,Makefile} $d/pkg/csrc/
    [ -n "$alt" ] && cp $alt $d/pkg/csrc/rq_kernels.cu
    make -s -C $d/pkg/csrc EXTRA="$f" OUT=$R/paper_1408_5526_b200/librqmc_b200_$n.so > $d/log 2>&1 || tail -20 $d/log
    grep -h "spill" $d/pkg/csrc/ptxas.log | sort | uniq -c | grep -v " 0 bytes spill stores" | sed "s/^/$n: /"
    rm -rf $d ) &
done
wait
ls -la $R/paper_1408_5526_b200/librqmc_b200_*.so
