timeout 900 python tools/c4_var.py random 4 2>&1 | tail -4
L0S_QR_SCREEN=tsqr timeout 900 python tools/c4_var.py random 3 2>&1 | tail -3
