# A/B sweep of the streaming-kernel knobs (env: VP, ring KB, slots per CTA); "0 0 0" = items_kernel
for cfg in "0 0 0" "1 48 128" "1 48 256" "1 32 128" "2 48 128" "2 48 256" "1 64 256"; do
  set -- $cfg
  if [ "$1" = "0" ]; then unset KLAY_STREAM; else export KLAY_STREAM=1; fi
  KLAY_STREAM_VP=$1 KLAY_STREAM_RING_KB=$2 KLAY_STREAM_SPC=$3 timeout 200 python bench.py --steps 20 --warmup 3 --no-extra --no-cpu-baseline --no-e2e --sustain 0 > gpurun_out/sw_$1_$2_$3.json 2>/dev/null
done
