for v in 3 2 1; do PBH_AB_OFF=$v timeout 900 python tools/probe_c4.py --ds "" --c1 1000000 2>&1 | grep cfg | sed "s/^/ab=$v /"; done
