# Record of a rejected experiment (profiles/r02/*_rejected.txt): its knob was removed with the code; see git history.
cd build/pairpkg
CKB_IMG_PAIR=1 timeout 300 python tools/shard_timing.py --worlds 8 --reps 5 2>&1 | tail -1
CKB_IMG_PAIR=1 timeout 600 ncu --set full --clock-control none --kernel-name-base function -k k_images_pair -s 3 -c 1 -o ../../gpurun_out/pair_w8 python tools/shard_timing.py --worlds 8 --reps 2 > /dev/null 2>&1; echo ncu=$?
