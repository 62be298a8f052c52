cd /root/repo
for v in _lib_keep _lib_o1; do echo "== $v"; HXG_PW=1 HXG_LIB=$PWD/paper_1711_00984_b200/$v/libhexgram_b200.so python tools/pw_diff.py --space H1 --p 7 | cut -c1-200; done
echo "== _lib (per-space WO)"; HXG_PW=1 python tools/pw_diff.py --space H1 --p 7 | cut -c1-200
python -m pytest tests -m gpu -q -x -k "high_order_general or sweep_high_order" 2>&1 | tail -1
for w in c5_hdiv_p8_general c5_hdiv_p9_general c5_hdiv_p10_general; do ELEM=256 bash tools/wl_quick.sh $w; HXG_PW=0 ELEM=256 bash tools/wl_quick.sh $w; done
