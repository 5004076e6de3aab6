# checking runs (compute-sanitizer is closed on this pool): the GPU suite with
#  (1) every scratch buffer poisoned on each fetch (CKB_POISON=1, graphs off), and
#  (2) additionally every kernel's dynamic shared memory poisoned at entry (build/variants/libpoison.so,
#      built by: python tools/build_variants.py poison=CKB_POISON_SMEM)
CKB_POISON=1 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/poison_global.txt 2>&1; echo global rc=$?; tail -3 gpurun_out/poison_global.txt
CKB_LIB=build/variants/libpoison.so CKB_POISON=1 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/poison_smem.txt 2>&1; echo smem rc=$?; tail -3 gpurun_out/poison_smem.txt
