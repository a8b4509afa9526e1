# GPU parity suite + DPD headline A/B of the current tree (VARIANTS env: extra builds)
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
VARIANTS="${VARIANTS:-}" NCU=1 bash tools/gpu_ms.sh
