for k in 0 512; do for w in planted random mt4; do echo "K'=$k $w"; L0S_KPRIME=$k timeout 900 python tools/c4_var.py $w 2 2>&1 | tail -2; done; done
