# sync-free SpTRSV: grid-size sweep (fewer spinning threads)
mkdir -p gpurun_out/sf
for g in 296 592 1184; do
GDSW_SF_GRID=$g timeout 300 python tools/profile_ts.py C2ilu 20 > gpurun_out/sf/ts_g$g.txt 2>&1; echo "grid $g: $(tail -1 gpurun_out/sf/ts_g$g.txt)"
done
