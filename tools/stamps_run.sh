for k in 2 3 4; do echo "== k=$k"; timeout 120 python tools/lu_stamps.py $k 2048 2>&1 | tail -22; done
