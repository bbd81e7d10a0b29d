# virtual-flavour A/B: exp/lib_base.so vs the in-tree build
for L in exp/lib_base.so paper_2504_18211_b200/libouro_b200.so; do
  n=$(basename $L .so)
  for c in vapq8g vlpq8g vacq8g vlcq8g; do
    OURO_B200_LIB=$PWD/$L timeout 300 python bench.py --config $c --sizes 16,1024,8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/abv_${n}_$c.json 2>/dev/null
  done
done
