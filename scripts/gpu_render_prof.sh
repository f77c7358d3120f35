# ncu launch lists of one render+resolve frame for c2 / c4 / the c5 per-GPU shard,
# with the L2 atomic / read counters of the keybuf fold (north_star: L2 atomic throughput)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_red.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sector_op_red_hit_rate.pct,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
B="--steps 1 --warmup 3 --no-e2e --no-cpu --no-pipeline --no-morton --no-gsplat --no-parity"
for w in c2 c4 c5; do
  P=""; [ $w = c5 ] && P="--points 250000000"
  timeout 600 ncu --metrics $M --clock-control none -k regex:"render|hiz|resolve" --csv --log-file gpurun_out/rprof_$w.csv python bench.py --workload $w $P $B > gpurun_out/rprof_$w.log 2>&1; echo "ncu $w rc=$?"
done
