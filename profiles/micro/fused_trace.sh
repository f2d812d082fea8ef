cd $GRAFT_REPO_ROOT
PI2_NVCC_EXTRA="-DPI2_TC_TRACE" python -c "from paper_1503_00330_b200 import _build; _build.build(force=True)" || exit 1
for c in C2 C4; do timeout 300 python profiles/micro/fused_trace.py --config $c; done
