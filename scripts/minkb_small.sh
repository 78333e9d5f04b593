export PYTHONUNBUFFERED=1
S="160 768 768;352 768 768;608 768 768;160 768 3072;352 768 3072;160 2304 768;160 3072 768;1216 768 768"
for mk in 8 6 4 3; do echo "== MINKB=$mk"; FTB_SPLIT_MINKB=$mk SHAPES="$S" timeout 200 python scripts/time_shapes.py; done 2>&1 | tee gpurun_out/minkb_small.txt
