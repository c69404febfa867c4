EBC200_LIB_PATH=paper_2105_12026_b200/libebc200_trace.so python tools/ub_trace.py C2 2>&1 | tail -1
EBC200_LIB_PATH=paper_2105_12026_b200/libebc200_trace.so python tools/ub_trace.py C4 2>&1 | tail -1
bash tools/gpu_iter_ub.sh
