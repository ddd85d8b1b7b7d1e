for v in w8 pxh pth pboth; do echo "== $v"; ZOLO_GMRES_LAG=0 ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so python tools/dev/probe_time.py cfg3 2>&1 | tail -1; done
