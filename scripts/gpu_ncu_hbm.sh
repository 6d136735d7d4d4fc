# ncu of the HBM-bound kernels on the final tree: merge/loss, gather, bookkeeping
# (one 16k-row micro-batch) and H1 over the whole 6.18M-row mini-batch.
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct"
timeout -s KILL 600 ncu --metrics $M --print-units base --csv -k regex:"k_merge|k_gather|k_flags|k_compact|k_scan|k_validate|k_stats|k_grpo" --log-file gpurun_out/ncu_hbm_mb.csv python scripts/probe.py --rows 16384 --reps 2 > /dev/null 2>&1; echo "mb rc=$?"
timeout -s KILL 600 ncu --metrics $M --print-units base --csv -k regex:"k_flags|k_compact|k_scan|k_validate" --log-file gpurun_out/ncu_hbm_h1.csv python scripts/probe_h1.py --reps 2 > /dev/null 2>&1; echo "h1 rc=$?"
