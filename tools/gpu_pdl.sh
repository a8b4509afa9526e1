timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
VARIANTS="nopdl" NCU=1 bash tools/gpu_ms.sh
