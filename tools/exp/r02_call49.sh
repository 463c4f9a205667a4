cd $GRAFT_REPO_ROOT
for et in 0 1; do for snr in -3 2.5; do
echo "== et=$et snr=$snr"
timeout 600 ncu --metrics smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:decode_pair16 -s 1 -c 1 --csv python tools/exp/fixed_one.py wifi 648 1/2 i16 $snr $et 2>&1 | grep -E "decode_pair16" | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done; done
