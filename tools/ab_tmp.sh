python tools/mlp_quick.py 606208 5 2>&1 | grep cfg
DFFM_LIB_PATH=build_var/tct/libdffm.so python tools/tc_trace.py cfg5 2>&1 | tail -11
timeout 600 python -m pytest tests/test_gpu_forward.py tests/test_gpu_quant_hash_ctx.py -q -x 2>&1 | tail -3
