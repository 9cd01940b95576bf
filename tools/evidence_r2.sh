# Round-2 evidence on one GPU box (run from the repo root): plain run first,
# then the ncu passes (one tool per gpurun call). Outputs in gpurun_out/.
set -x
python tools/ncu_target.py 1 > gpurun_out/plain.log 2>&1 || exit 1
# every launch of one fwd+bwd step (config C, B = 1024): time + DRAM bytes
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r2_launches.csv python tools/ncu_target.py 1 > gpurun_out/ncu_list.log 2>&1
# full captures: the forward log-sum-exp class (layer 10) and the dominant
# class, the backward pass-through with route masks (layer 9)
ncu --set full --clock-control none --import-source on -k "regex:items_kernel<float, 4" -s 4 -c 1 \
    -o gpurun_out/r2_fwd_lse10 python tools/ncu_target.py 1 > gpurun_out/ncu_lse.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:BwdGather<float, 3>" -s 15 -c 1 \
    -o gpurun_out/r2_bwd_passa9 python tools/ncu_target.py 1 > gpurun_out/ncu_passa.log 2>&1
# the opt-in streaming kernel on the same forward product layer 9
KLAY_STREAM=1 python tools/ncu_target.py 1 > gpurun_out/plain_stream.log 2>&1 && \
KLAY_STREAM=1 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 8 -c 1 \
    -o gpurun_out/r2_stream_fwd9 python tools/ncu_target.py 1 > gpurun_out/ncu_stream.log 2>&1
echo done
