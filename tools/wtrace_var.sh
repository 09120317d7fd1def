cp paper_2510_05885_b200/libncl_b200.so /tmp/orig.so
cp _var/trace.so paper_2510_05885_b200/libncl_b200.so
bash tools/wtrace.sh
cp /tmp/orig.so paper_2510_05885_b200/libncl_b200.so
bash tools/variants.sh
