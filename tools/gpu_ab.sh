# A/B: abtest/lib_a.so vs abtest/lib_b.so on the same box, alternating
mkdir -p gpurun_out
for r in 1 2; do
  for v in a b; do
    RAMA_LIB=$PWD/abtest/lib_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$r.log 2>&1
  done
done
