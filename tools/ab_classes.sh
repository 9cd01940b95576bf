# A/B of abvar/base vs the in-tree library on several configs (class breakdown)
for v in base new; do
  if [ $v = base ]; then export KLAY_LIB=$PWD/abvar/base/libklay.so; else unset KLAY_LIB; fi
  for a in "E float64 128" "B float64 256" "C float32 128" "C float32 1024"; do
    echo "== $v $a"; python tools/class_breakdown.py $a | head -1
  done
done
