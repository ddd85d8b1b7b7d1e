mkdir -p gpurun_out/s5
# trailing kernel of the left-looking factorization: a mid-tree launch and a top-of-tree launch of pole 0
ncu --set full --clock-control none --import-source on -k regex:trailing_level -s 60 -c 2 -o gpurun_out/s5/trailing_mid python tools/dev/factor_only.py cfg3 > gpurun_out/s5/ncu_trailing_mid.log 2>&1
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"trailing_level|diag_level|panel_level|scale_sp|swizzle|tile_mask|tile_work|scatter_sp" -c 6000 --csv --log-file gpurun_out/s5/factor_launches.csv python tools/dev/factor_only.py cfg3 1 > gpurun_out/s5/ncu_factor_list.log 2>&1
tail -3 gpurun_out/s5/ncu_factor_list.log
