OUT=gpurun_out/r2bj_sanitize.txt bash scripts/sanitize_paths.sh > /dev/null 2>&1
cat gpurun_out/r2bj_sanitize.txt
SEEDS=500:700 timeout 1500 python scripts/fuzz_campaign.py > gpurun_out/r2bj_fuzz.txt 2>&1; echo fuzz_rc=$?
LARGE=1 SEEDS=500:580 timeout 1500 python scripts/fuzz_campaign.py > gpurun_out/r2bj_fuzz_large.txt 2>&1; echo fuzz_large_rc=$?
tail -3 gpurun_out/r2bj_fuzz.txt gpurun_out/r2bj_fuzz_large.txt
