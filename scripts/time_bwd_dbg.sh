for D in 0 1 2 4 5 7; do echo "DBG=$D"; MOBA_BWD_DBG=$D IMPLS=tc python scripts/time_bwd.py 2>&1 | grep atomic; done
