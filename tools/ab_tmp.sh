for g in 148 128 112 96; do echo "== gather grid $g"; DFFM_RSW_GRID=$g python tools/mlp_quick.py 606208 5 2>&1 | grep cfg; done
