# sort-reduce huge-row threshold variants on c2 / c3 / c4
VARIANTS="base abtest/huge256/librama_b200.so abtest/huge128/librama_b200.so" WL="c2 c3" STEPS=8 bash tools/gpu_ab.sh
