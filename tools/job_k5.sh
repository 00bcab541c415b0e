set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/diag_k5.py 100000 100 30
SLQ_L2_KEEP_MB=0 python tools/diag_k5.py 100000 100 30
SLQ_NO_FUSED_K5=1 SLQ_L2_KEEP_MB=0 python tools/diag_k5.py 100000 100 30
python tools/diag_k5.py 200000 100 30
SLQ_L2_KEEP_MB=0 python tools/diag_k5.py 200000 100 30
