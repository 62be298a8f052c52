cd /root/repo
for v in _lib_rj4 _lib_ctw; do echo "== $v"; HXG_PW=1 HXG_LIB=$PWD/paper_1711_00984_b200/$v/libhexgram_b200.so python tools/pw_diff.py --space H1 --p 7 | cut -c1-150; done
