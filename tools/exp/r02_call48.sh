cd $GRAFT_REPO_ROOT
for et in 0 1; do for snr in -3 2.5; do
timeout 600 ncu --metrics smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:decode_pair16 -s 1 -c 1 --csv python tools/exp/fixed_one.py wifi 648 1/2 i16 $snr $et 2>&1 | grep -E "decode_pair16|dB et" | awk -F'","' '{print $NF, $(NF-2)}' | tr -d '"' | tr '\n' ' '; echo " <- et=$et snr=$snr"
done; done
for code in "wifi 648 1/2" "wifi 648 5/6" "wimax 672 1/2" "wimax 768 3/4A" "wifi 1296 1/2"; do for et in 0 1; do python tools/exp/fixed_one.py $code i16 2.5 $et; done; done
