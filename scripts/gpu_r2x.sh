SHAPES="dense 16 4096 4096;dense 256 4096 4096;dense 608 768 768;dense 1024 768 3072;bmm 384 100 100 64 nk;bmm 384 46 46 64 nk" python scripts/prof_chain.py 2>&1 | tail -30
