# one GPU iteration: quick parity subset, streaming-launch traces, the bench
# line without the extra configs (run from the repo root on the GPU box)
timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_engine.log 2>&1
echo "engine tests rc=$?"
tail -2 gpurun_out/t_engine.log
bash tools/stream_trace.sh > gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --no-cpu-baseline --no-e2e --sustain 0 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
