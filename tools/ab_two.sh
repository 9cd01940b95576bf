# A/B: the in-tree libklay.so against abvar/base/libklay.so (bench C, B = 1024 and 128)
for b in 1024 128; do
  for v in base new; do
    if [ $v = base ]; then export KLAY_LIB=$PWD/abvar/base/libklay.so; else unset KLAY_LIB; fi
    timeout 200 python bench.py --batch $b --steps 30 --warmup 3 --no-extra --no-cpu-baseline --no-e2e --sustain 0 > gpurun_out/ab_${v}_$b.json 2>/dev/null
  done
done
