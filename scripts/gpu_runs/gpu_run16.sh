cd $GRAFT_REPO_ROOT
for mode in "" "--serial"; do
timeout 900 python scripts/c3_run.py --policy cfs-peer --proxy-gb 16 $mode > gpurun_out/r01_c3_overlap$mode.json 2> gpurun_out/r01_c3_overlap$mode.err; echo "overlap $mode $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_overlap$mode.json')); print(d['streams'], 'wall', d['wall_s'], 'swapms', d['swap_device_ms'], d['verify_mismatches'])"; tail -n 2 gpurun_out/r01_c3_overlap$mode.err
done
for mode in "" "--serial"; do
timeout 900 python scripts/c3_run.py --policy cfs-host --proxy-gb 16 $mode > gpurun_out/r01_c3_overlap_host$mode.json 2> gpurun_out/r01_c3_overlap_host$mode.err; echo "overlap host $mode $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_overlap_host$mode.json')); print(d['streams'], 'wall', d['wall_s'], 'swapms', d['swap_device_ms'], d['verify_mismatches'])"
done
