/* Host side of the event log: device co_event records -> the reference's
 * event dicts (engine.py:353 arrive, :520 admit, :630-633 iter, :383-384
 * preempt, :401-402 readmit, :412 complete), built with the CPython C API.
 * Engine.events calls it once per drain; in Python the same conversion cost
 * more than the scheduler step itself on the per-step API path.
 *
 *   _hostlog.convert(events_addr, n, members_addr, rid_list, strategy_names, cause_names) -> list
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef struct {  /* include/cacheopt.h co_event */
    int32_t kind, idx;
    int64_t t, a, b, c;
} co_event;

enum { EV_ARRIVE = 0, EV_ADMIT = 1, EV_ITER = 2, EV_PREEMPT = 3, EV_READMIT = 4, EV_COMPLETE = 5 };

static PyObject *k_ev, *k_t, *k_req, *k_end, *k_tokens, *k_members, *k_strategy, *k_kv, *k_cause, *k_ready_at;
static PyObject *v_arrive, *v_admit, *v_iter, *v_preempt, *v_readmit, *v_complete;

static int set_steal(PyObject *d, PyObject *k, PyObject *v) {
    if (!v) return -1;
    int r = PyDict_SetItem(d, k, v);
    Py_DECREF(v);
    return r;
}

static PyObject *convert(PyObject *self, PyObject *args) {
    unsigned long long ev_addr, mem_addr;
    Py_ssize_t n;
    PyObject *rid, *strat, *cause;
    if (!PyArg_ParseTuple(args, "KnKO!O!O!", &ev_addr, &n, &mem_addr, &PyList_Type, &rid, &PyTuple_Type, &strat,
                          &PyTuple_Type, &cause))
        return NULL;
    const co_event *ev = (const co_event *)(uintptr_t)ev_addr;
    const int32_t *mem = (const int32_t *)(uintptr_t)mem_addr;
    const Py_ssize_t nrid = PyList_GET_SIZE(rid);
    PyObject *out = PyList_New(n);
    if (!out) return NULL;
    for (Py_ssize_t k = 0; k < n; k++) {
        const co_event *e = ev + k;
        PyObject *d = PyDict_New();
        if (!d) goto fail;
        PyList_SET_ITEM(out, k, d);
        if (e->idx < 0 || (e->kind != EV_ITER && e->idx >= nrid)) {
            PyErr_SetString(PyExc_ValueError, "event index out of range");
            goto fail;
        }
        PyObject *req = e->kind == EV_ITER ? NULL : PyList_GET_ITEM(rid, e->idx);
        switch (e->kind) {
            case EV_ITER: {
                if (PyDict_SetItem(d, k_ev, v_iter) || set_steal(d, k_t, PyLong_FromLongLong(e->t)) ||
                    set_steal(d, k_end, PyLong_FromLongLong(e->a)) ||
                    set_steal(d, k_tokens, PyLong_FromLongLong(e->b)))
                    goto fail;
                const Py_ssize_t m = e->idx;
                const int32_t *p = mem + 2 * e->c;
                PyObject *ms = PyList_New(m);
                if (!ms) goto fail;
                for (Py_ssize_t j = 0; j < m; j++) {
                    const int32_t i = p[2 * j];
                    if (i < 0 || i >= nrid) {
                        Py_DECREF(ms);
                        PyErr_SetString(PyExc_ValueError, "member index out of range");
                        goto fail;
                    }
                    PyObject *pair = PyList_New(2);
                    PyObject *tok = PyLong_FromLong(p[2 * j + 1]);
                    if (!pair || !tok) {
                        Py_XDECREF(pair);
                        Py_XDECREF(tok);
                        Py_DECREF(ms);
                        goto fail;
                    }
                    PyObject *r = PyList_GET_ITEM(rid, i);
                    Py_INCREF(r);
                    PyList_SET_ITEM(pair, 0, r);
                    PyList_SET_ITEM(pair, 1, tok);
                    PyList_SET_ITEM(ms, j, pair);
                }
                if (set_steal(d, k_members, ms)) goto fail;
                break;
            }
            case EV_ARRIVE:
            case EV_ADMIT:
            case EV_COMPLETE:
                if (PyDict_SetItem(d, k_ev, e->kind == EV_ARRIVE ? v_arrive : e->kind == EV_ADMIT ? v_admit
                                                                                                   : v_complete) ||
                    set_steal(d, k_t, PyLong_FromLongLong(e->t)) || PyDict_SetItem(d, k_req, req))
                    goto fail;
                break;
            case EV_PREEMPT:
                if (e->b < 0 || e->b >= PyTuple_GET_SIZE(strat) || e->c < 0 || e->c >= PyTuple_GET_SIZE(cause)) {
                    PyErr_SetString(PyExc_ValueError, "preempt event code out of range");
                    goto fail;
                }
                if (PyDict_SetItem(d, k_ev, v_preempt) || set_steal(d, k_t, PyLong_FromLongLong(e->t)) ||
                    PyDict_SetItem(d, k_req, req) || PyDict_SetItem(d, k_strategy, PyTuple_GET_ITEM(strat, e->b)) ||
                    set_steal(d, k_kv, PyLong_FromLongLong(e->a)) ||
                    PyDict_SetItem(d, k_cause, PyTuple_GET_ITEM(cause, e->c)))
                    goto fail;
                break;
            case EV_READMIT:
                if (PyDict_SetItem(d, k_ev, v_readmit) || set_steal(d, k_t, PyLong_FromLongLong(e->t)) ||
                    PyDict_SetItem(d, k_req, req) || set_steal(d, k_ready_at, PyLong_FromLongLong(e->a)))
                    goto fail;
                break;
            default:
                PyErr_SetString(PyExc_ValueError, "unknown event kind");
                goto fail;
        }
    }
    return out;
fail:
    Py_DECREF(out);
    return NULL;
}

static PyMethodDef methods[] = {
    {"convert", convert, METH_VARARGS, "co_event records -> the reference's event dicts"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_hostlog", NULL, -1, methods};

PyMODINIT_FUNC PyInit__hostlog(void) {
#define S(var, text) if (!(var = PyUnicode_InternFromString(text))) return NULL;
    S(k_ev, "ev") S(k_t, "t") S(k_req, "req") S(k_end, "end") S(k_tokens, "tokens") S(k_members, "members")
    S(k_strategy, "strategy") S(k_kv, "kv") S(k_cause, "cause") S(k_ready_at, "ready_at")
    S(v_arrive, "arrive") S(v_admit, "admit") S(v_iter, "iter") S(v_preempt, "preempt") S(v_readmit, "readmit")
    S(v_complete, "complete")
#undef S
    return PyModule_Create(&mod);
}
