# NVTX ranges of the C ABI: each ncu --nvtx-include filter must select exactly its stage kernel (prints 1, 0, 1)
cd $GRAFT_REPO_ROOT
ncu --nvtx --nvtx-include "lwpr/" --metrics gpu__time_duration.sum --csv python profiles/profile_step.py --iters 1 2>/dev/null | grep -c "lwpr_tc_kernel"
ncu --nvtx --nvtx-include "lwpr/" --metrics gpu__time_duration.sum --csv python profiles/profile_step.py --iters 1 2>/dev/null | grep -c "rollout_group_kernel"
ncu --nvtx --nvtx-include "partials/" --metrics gpu__time_duration.sum --csv python profiles/profile_step.py --iters 1 2>/dev/null | grep -c "partials_kernel"
