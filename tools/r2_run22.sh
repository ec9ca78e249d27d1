for th in 8 12 16; do L0S_COPY_THREADS=$th timeout 300 python tools/e2e_probe.py 2>&1 | grep pageable | tail -2 | sed "s/^/threads $th: /"; done
timeout 300 python tools/e2e_probe.py 2>&1 | tail -12
