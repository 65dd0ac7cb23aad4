# width-512 tensor-core MLP: first run on the debug-wait build (mbarrier timeouts trap instead of hanging)
SWR_LIB=tools/libswr_widedbg.so timeout -s KILL 400 python -m pytest tests/test_mlp_wide.py -x -q --timeout 300 2>&1 | tail -25
