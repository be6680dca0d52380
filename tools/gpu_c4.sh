# C4: staging-buffer count sweep of the index kernel (warps per SM follow from shared memory)
for s in 2 4 8; do echo stages=$s; BR_SHUFFLE_KERNEL=idx BR_IDX_STAGES=$s REPS=10 python tools/shuffle_time.py c4 idx; done
