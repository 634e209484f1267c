python tools/trace_chunks.py > gpurun_out/trace.log 2>&1
CM_TMEM=0 python tools/trace_chunks.py > gpurun_out/trace_tm0.log 2>&1
