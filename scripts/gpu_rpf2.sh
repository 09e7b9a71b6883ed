cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/gpu_env_ab.sh rpf2 GNNCG_GAT_RPF "1 0" 2 --no-ncu --no-parity
for v in 1 0; do GNNCG_GAT_RPF=$v timeout 600 ncu --section LaunchStats --section Occupancy --section SpeedOfLight --metrics dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gat_bwd_src_lean -c 1 --csv --log-file gpurun_out/ncu_rpf_$v.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > /dev/null 2>&1; done
