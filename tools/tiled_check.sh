set -x
VOXSCHUR_TILED=1 timeout 300 python tools/prof_inner.py C1 1 --no-phases 2>&1 | tail -3
VOXSCHUR_TILED=1 timeout 300 python tools/prof_inner.py C2 1 --no-phases 2>&1 | tail -3
VOXSCHUR_CG=1 timeout 300 python tools/prof_inner.py C2 1 --no-phases 2>&1 | tail -3
VOXSCHUR_TILED=1 timeout 600 python -m pytest tests/test_gpu_scale.py -x -q 2>&1 | tail -5
