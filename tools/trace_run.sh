# CTA timelines of K3 (mode 3) and the fused pass (mode 9) at J = 12 and J = 1 (needs variants/trace.so, a -DNLV_TRACE build)
cp paper_1301_1215_b200/libnlinv.so /tmp/base.so
cp paper_1301_1215_b200/variants/trace.so paper_1301_1215_b200/libnlinv.so
for J in 12 1; do for m in 3 9; do echo "== J=$J mode $m"; J=$J timeout 120 python tools/trace_cta.py $m 2>&1 | tail -10; done; done
cp /tmp/base.so paper_1301_1215_b200/libnlinv.so
