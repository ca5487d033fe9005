for v in hl hf; do echo "== $v"; DFFM_LIB_PATH=build_var/$v/libdffm.so python tools/mlp_quick.py 2097152 3 2>&1 | grep cfg; done
python tools/mlp_quick.py 2097152 3 2>&1 | grep cfg
