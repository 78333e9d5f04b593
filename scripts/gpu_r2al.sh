SHAPES="dense 4096 3072 768;dense 4096 4096 4096" python scripts/prof_chain.py 2>&1 | tail -8
FTB_PAIR=1 SHAPES="dense 4096 3072 768;dense 4096 4096 4096" python scripts/prof_chain.py 2>&1 | tail -8
