# L2->SM bandwidth hypothesis: TMA micro (L2-resident and HBM-streaming), big Dense single vs CTA pair,
# ncu L2 counters of one big launch each way
./scripts/micro/tma_bench > gpurun_out/r2aq_tma_bench.txt 2>&1
S="dense 4096 3072 768;dense 4096 2304 768;dense 4096 768 3072;dense 1536 3072 768;dense 4096 4096 4096;dense 8192 8192 8192"
SHAPES="$S" NL=4 python scripts/chain_time.py > gpurun_out/r2aq_chain.txt 2>&1
SHAPES="$S" NL=4 FTB_PAIR=1 python scripts/chain_time.py >> gpurun_out/r2aq_chain.txt 2>&1
TAG=single python scripts/step_time.py >> gpurun_out/r2aq_chain.txt 2>&1
TAG=pair FTB_PAIR=1 python scripts/step_time.py >> gpurun_out/r2aq_chain.txt 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum.per_second
for P in 0 1; do
SHAPES="dense 4096 3072 768;dense 4096 4096 4096" NL=1 COLD=0 FTB_PAIR=$P timeout 600 ncu --metrics $M --clock-control none -k regex:ftb_ -s 2 -c 4 --csv --log-file gpurun_out/r2aq_ncu_p$P.csv python scripts/chain_time.py > gpurun_out/r2aq_ncu_p$P.log 2>&1
done
cat gpurun_out/r2aq_tma_bench.txt gpurun_out/r2aq_chain.txt
