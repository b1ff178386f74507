python tools/sort_probe.py 28
for v in t256i16m3 t512i8m3 t256i24m2 t512i16m1; do echo $v; PASGAL_BCC_LIB=paper_2404_17101_b200/lib/variants/lib_$v.so python tools/sort_probe.py 28; done
