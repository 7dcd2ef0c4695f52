# Interleaved A/B over library variants: LIBS="v000 v111 ..." ROUNDS=2 bash tools/gpu_ab2.sh "<bench args>" ...
rm -f gpurun_out/ab2.json
for r in $(seq ${ROUNDS:-2}); do
for args in "$@"; do
  for v in $LIBS; do
    RQMC_B200_LIB=$PWD/paper_1408_5526_b200/librqmc_b200_$v.so timeout 300 python bench.py $args --no-cpu-baseline --steps ${STEPS:-3} 2>>gpurun_out/ab2.err | sed "s|^{|{\"lib\": \"$v\", \"args\": \"$args\", |" >> gpurun_out/ab2.json
  done
done
done
python tools/ab_table.py gpurun_out/ab2.json
