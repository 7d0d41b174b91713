run() { timeout 300 "$@" 2>&1 | grep '^{' ; }
for c in 8 6; do echo "base ctas=$c"; BCSS_SYM_CTAS=$c run python tools/sym_upload_timing.py 5 --steps 8; done
for c in 8 6 4; do echo "t1024u6 ctas=$c"; BCSS_SYM_CTAS=$c run python tools/variant.py t1024u6 tools/sym_upload_timing.py 5 --steps 8; done
