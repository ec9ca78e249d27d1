timeout 900 python tools/c4_var.py mt4 5 2>&1 | tail -5
L0S_QR_SCREEN=tsqr timeout 900 python tools/c4_var.py mt4 4 2>&1 | tail -4
timeout 900 python tools/c4_var.py random 5 2>&1 | tail -5
