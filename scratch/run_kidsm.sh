CMD="python bench.py --workload kidnap --steps 2 --warmup 25 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_smooth_round" -s 300 -c 10 --csv $CMD > gpurun_out/kidsm.csv 2> gpurun_out/kidsm.err; echo "rc=$?"
