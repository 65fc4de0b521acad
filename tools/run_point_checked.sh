# The degenerate point cloud through the forced spread path: release build,
# then the bounds-checked builds (tools/build_variant.py check / check2 first).
python -c "from paper_2302_00942_b200 import build; build.build()" >/dev/null 2>&1
cp paper_2302_00942_b200/lib/librfd.so /tmp/librfd_release.so
echo "== release"; timeout 300 python tools/point_case.py 2>&1 | grep -v "^  " | head -12
echo "== release, no sync check"; RFD_SYNC_CHECK=0 timeout 300 python tools/point_case.py 2>&1 | grep -v "^  " | head -6
for v in check; do
  echo "== $v"; cp abtest/$v/librfd.so paper_2302_00942_b200/lib/librfd.so
  timeout 300 python tools/point_case.py 2>&1 | grep -v Traceback | head -12
done
cp /tmp/librfd_release.so paper_2302_00942_b200/lib/librfd.so
