S="bmm 384 27 27 64 nk;bmm 384 46 46 64 nk;bmm 384 81 81 64 nk;bmm 384 100 100 64 nk;bmm 384 119 119 64 nk;bmm 1024 257 257 64 nk;dense 608 768 768"
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_prev.so python scripts/chain_time.py 2>&1 | cut -c 1-62
SHAPES="$S" python scripts/chain_time.py 2>&1 | cut -c 1-62
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
