# A/B of libklay variants under abvar/<name>/libklay.so (bench C at the given batches)
# usage: bash tools/ab_variants.sh "1024 128" base f16 b16 ...
batches=$1; shift
for b in $batches; do
  for v in "$@"; do
    KLAY_LIB=$PWD/abvar/$v/libklay.so timeout 200 python bench.py --batch $b --steps 30 --warmup 3 --no-extra --no-cpu-baseline --no-e2e --sustain 0 > gpurun_out/ab_${v}_$b.json 2>/dev/null
  done
done
