mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
RFD_SMALL_TRACE=1 python tools/small_trace.py 4 2>&1 | tail -12
python tools/graph_small.py 2>&1 | tail -8
RFD_NARROW=0 python tools/graph_small.py 2>&1 | tail -8
