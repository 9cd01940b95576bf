# per-CTA timing of single streaming launches (debug build, see klay.cu stream_trace_dump); build it first:
#   python -c "import __graft_entry__ as g; g.build(extra=['-DKLAY_STREAM_TRACE'], out='paper_2410_11415_b200/libklay_trace.so')"
export KLAY_LIB=$PWD/paper_2410_11415_b200/libklay_trace.so KLAY_STREAM=1 KLAY_STREAM_VP=1 KLAY_STREAM_SPC=128
for spec in "9 0" "10 0" "9 1" "10 1"; do
  set -- $spec
  KLAY_STREAM_TRACE_LAYER=$1 KLAY_STREAM_TRACE_DIR=$2 python tools/ncu_target.py 2 2>&1 | grep "stream trace"
done
