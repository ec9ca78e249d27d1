for k in 0 256 512 1024; do echo "K'=$k"; L0S_KPRIME=$k timeout 600 python tools/c4_once.py 2>&1 | cut -c1-420;
 L0S_KPRIME=$k L0S_TUNE_Y=planted timeout 600 python tools/tune_fit.py one 2>&1 | cut -c1-200; L0S_KPRIME=$k L0S_TUNE_Y=random timeout 600 python tools/tune_fit.py one 2>&1 | cut -c1-200; done
