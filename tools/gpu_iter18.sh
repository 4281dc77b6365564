set -x
for ty in 16 32; do OOCS_STEP_TY=$ty python tools/step_micro.py 2>&1 | tail -4; done
OOCS_STEP_TY=32 python -m pytest tests/test_gpu_parity.py -q -x -k "stencil or identity" 2>&1 | tail -2
