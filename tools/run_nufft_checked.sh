# Spread-path GPU tests against a build with the k_nufft.cu bounds checks
# (tools/build_variant.py check -DRFD_NUFFT_CHECK k_nufft.cu first).
python -c "from paper_2302_00942_b200 import build; build.build()" >/dev/null 2>&1
cp paper_2302_00942_b200/lib/librfd.so /tmp/librfd_release.so
cp abtest/check/librfd.so paper_2302_00942_b200/lib/librfd.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -m gpu -k "spread or gfi or sharded or config5_full or degenerate" ${1:+-k "$1"} 2>&1 | grep -E "passed|failed|FAILED|nufft check|Error|^E " | head -30
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
cp /tmp/librfd_release.so paper_2302_00942_b200/lib/librfd.so
