# Round-2 --set full captures (items_kernel launch indices from the launch
# list: 11 = the longest forward log-sum-exp launch, 85 = the longest
# backward pass-through-with-masks launch, 84 = the longest log-sum backward)
python tools/ncu_target.py 1 > gpurun_out/plain.log 2>&1 || exit 1
for spec in "11 r2_fwd_lse" "85 r2_bwd_passa" "84 r2_bwd_logsum" "8 r2_fwd_prod"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:items_kernel -s $1 -c 1 \
      -o gpurun_out/$2 python tools/ncu_target.py 1 > gpurun_out/ncu_$2.log 2>&1
done
echo done
