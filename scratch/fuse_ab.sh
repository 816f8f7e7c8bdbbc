python scratch/levels.py --tag fuse0 2>&1 | tail -1
FT_NO_FUSE0=1 python scratch/levels.py --tag nofuse 2>&1 | tail -1
FT_LEAF_DBG=4 python scratch/leafclk.py
