OUT=gpurun_out/r2bt_sanitize.txt bash scripts/sanitize_paths.sh > /dev/null 2>&1
cat gpurun_out/r2bt_sanitize.txt
SEEDS=700:900 timeout 1500 python scripts/fuzz_campaign.py > gpurun_out/r2bt_fuzz.txt 2>&1; echo fuzz_rc=$?
LARGE=1 SEEDS=700:780 timeout 1500 python scripts/fuzz_campaign.py > gpurun_out/r2bt_fuzz_large.txt 2>&1; echo fuzz_large_rc=$?
tail -n 2 gpurun_out/r2bt_fuzz.txt; tail -n 2 gpurun_out/r2bt_fuzz_large.txt
