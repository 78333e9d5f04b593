OUT=gpurun_out/r2ai_sanitize.txt bash scripts/sanitize_paths.sh > /dev/null 2>&1
echo "== memcheck: split-K concurrency (occupier) test" >> gpurun_out/r2ai_sanitize.txt
cat gpurun_out/r2ai_sanitize.txt
SEEDS=300:500 timeout 1500 python scripts/fuzz_campaign.py > gpurun_out/r2ai_fuzz.txt 2>&1; echo fuzz_rc=$?
LARGE=1 SEEDS=300:380 timeout 1500 python scripts/fuzz_campaign.py > gpurun_out/r2ai_fuzz_large.txt 2>&1; echo fuzz_large_rc=$?
tail -3 gpurun_out/r2ai_fuzz.txt gpurun_out/r2ai_fuzz_large.txt
