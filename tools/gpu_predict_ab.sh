# A/B of the drop-in predict(X) host pipeline (VKM_TRACE stage times) and the other host-staged calls.
for wc in 1 0 1 0; do
echo "wc=$wc"; VKM_HOUT_WC=$wc VKM_TRACE=1 python tools/trace_predict.py 2>&1 | tail -2
VKM_HOUT_WC=$wc python tools/prof_predict.py 2>&1 | grep -E "predict|encode"
done
