/* kr_pack.c -- host runtime: pack reference-shaped planning objects into the
 * fleet structure-of-arrays in native code.
 *
 * plan() (scheduler.py:254-276 in the reference) is called by the simulator
 * on every planning event with tens to thousands of pending requests; the
 * objects' fields and histories (PendingRequest, TaskState: core.py:132-249)
 * must be walked on the host every call.  Done in Python that walk is most of
 * a small plan's latency; this CPython extension does it in one pass of C and
 * writes the columns straight into the caller's mapped pinned arena, which
 * kr_plan_small (or kr_urgency) then reads over PCIe.
 *
 *   _kr_pack.pack(reqs, states, rank_of, host_addr, capacity, out_bytes)
 *       -> (osl, o32, oout, nsl)  offsets of the slot and int32 blocks and of
 *                                 the output region; or None when `capacity`
 *                                 bytes are not enough (the caller grows the
 *                                 arena and calls again)
 *
 * Layout at host_addr (each block 256-byte aligned):
 *   int64 [5][n]   t_start, issued_at, obs_captured_at, accum_gen, hist_off
 *   int64 [nsl][4] (gen_start, gen_end, exec_start, exec_end) per recorded
 *                  round, CSR by hist_off; max(n_gen, n_exec) rows a request,
 *                  an in-flight generation's end (None) and the shorter side's
 *                  padding stored as 0 (fleet.host_soa)
 *   int32 [5][n]   remaining, lexrank, skipped, n_exec, n_gen
 *   output region  out_bytes
 * Any attribute / lookup / conversion error propagates as the Python
 * exception (AttributeError, KeyError, TypeError, OverflowError). */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

static PyObject *s_task_id, *s_gen_starts, *s_gen_ends, *s_exec_intervals, *s_t_start,
    *s_issued_at, *s_obs_captured_at, *s_accumulated_generation, *s_last_exec_info,
    *s_remaining_actions, *s_skipped, *s_start, *s_end, *s_dict, *s_dc_fields;

static size_t align256(size_t b) { return (b + 255) / 256 * 256; }

/* int attribute of obj as int64 (new reference released here) */
static int attr_i64(PyObject* obj, PyObject* name, int64_t* out) {
    PyObject* v = PyObject_GetAttr(obj, name);
    if (!v) return -1;
    long long x = PyLong_AsLongLong(v);
    Py_DECREF(v);
    if (x == -1 && PyErr_Occurred()) return -1;
    *out = (int64_t)x;
    return 0;
}

static int to_i32(int64_t v, int32_t* out) {
    if (v < INT32_MIN || v > INT32_MAX) {
        PyErr_SetString(PyExc_OverflowError, "value does not fit the fleet's int32 column");
        return -1;
    }
    *out = (int32_t)v;
    return 0;
}

/* The three history sequences of a task state (new references). */
static int history(PyObject* st, PyObject** g, PyObject** ge, PyObject** ex) {
    *g = *ge = *ex = NULL;
    PyObject* a = PyObject_GetAttr(st, s_gen_starts);
    if (!a) return -1;
    *g = PySequence_Fast(a, "gen_starts must be a sequence");
    Py_DECREF(a);
    if (!*g) return -1;
    a = PyObject_GetAttr(st, s_gen_ends);
    if (!a) return -1;
    *ge = PySequence_Fast(a, "gen_ends must be a sequence");
    Py_DECREF(a);
    if (!*ge) return -1;
    a = PyObject_GetAttr(st, s_exec_intervals);
    if (!a) return -1;
    *ex = PySequence_Fast(a, "exec_intervals must be a sequence");
    Py_DECREF(a);
    return *ex ? 0 : -1;
}

static PyObject* pack(PyObject* self, PyObject* args) {
    PyObject *reqs_in, *states, *rank_of;
    unsigned long long addr;
    Py_ssize_t capacity, out_bytes;
    if (!PyArg_ParseTuple(args, "OOOKnn", &reqs_in, &states, &rank_of, &addr, &capacity,
                          &out_bytes))
        return NULL;
    PyObject* reqs = PySequence_Fast(reqs_in, "reqs must be a sequence");
    if (!reqs) return NULL;
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(reqs);
    PyObject** R = PySequence_Fast_ITEMS(reqs);
    PyObject** S = PyMem_Malloc(sizeof(PyObject*) * (size_t)(n > 0 ? n : 1));
    if (!S) {
        Py_DECREF(reqs);
        return PyErr_NoMemory();
    }
    Py_ssize_t i, got = 0;
    PyObject* result = NULL;
    /* pass 1: states and slot counts */
    size_t nsl = 0;
    for (i = 0; i < n; i++, got++) {
        PyObject* tid = PyObject_GetAttr(R[i], s_task_id);
        if (!tid) goto done;
        S[i] = PyObject_GetItem(states, tid);
        Py_DECREF(tid);
        if (!S[i]) goto done;
        PyObject *g, *ge, *ex;
        if (history(S[i], &g, &ge, &ex)) {
            Py_XDECREF(g); Py_XDECREF(ge); Py_XDECREF(ex);
            got++;
            goto done;
        }
        Py_ssize_t lg = PySequence_Fast_GET_SIZE(g), le = PySequence_Fast_GET_SIZE(ex);
        nsl += (size_t)(lg > le ? lg : le);
        Py_DECREF(g); Py_DECREF(ge); Py_DECREF(ex);
    }
    {
        const size_t nslot = nsl > 0 ? nsl : 1;
        const size_t osl = align256(40 * (size_t)n);
        const size_t o32 = osl + align256(32 * nslot);
        const size_t oout = o32 + align256(20 * (size_t)n);
        if (oout + (size_t)out_bytes > (size_t)capacity) {
            result = Py_None;
            Py_INCREF(result);
            goto done;
        }
        unsigned char* base = (unsigned char*)(uintptr_t)addr;
        int64_t* c64 = (int64_t*)base;
        int64_t* sl = (int64_t*)(base + osl);
        int32_t* c32 = (int32_t*)(base + o32);
        if (nsl == 0) memset(sl, 0, 32);
        /* pass 2: the columns */
        int64_t off = 0;
        for (i = 0; i < n; i++) {
            PyObject *r = R[i], *st = S[i];
            int64_t v;
            int32_t v32;
            if (attr_i64(st, s_t_start, &c64[i])) goto done;
            if (attr_i64(r, s_issued_at, &c64[n + i])) goto done;
            if (attr_i64(r, s_obs_captured_at, &c64[2 * n + i])) goto done;
            if (attr_i64(st, s_accumulated_generation, &c64[3 * n + i])) goto done;
            c64[4 * n + i] = off;
            PyObject* lei = PyObject_GetAttr(r, s_last_exec_info);
            if (!lei) goto done;
            int rc = attr_i64(lei, s_remaining_actions, &v);
            Py_DECREF(lei);
            if (rc || to_i32(v, &c32[i])) goto done;
            PyObject* tid = PyObject_GetAttr(r, s_task_id);
            if (!tid) goto done;
            PyObject* rk = PyObject_GetItem(rank_of, tid);
            Py_DECREF(tid);
            if (!rk) goto done;
            long long x = PyLong_AsLongLong(rk);
            Py_DECREF(rk);
            if ((x == -1 && PyErr_Occurred()) || to_i32(x, &c32[n + i])) goto done;
            if (attr_i64(r, s_skipped, &v) || to_i32(v, &v32)) goto done;
            c32[2 * n + i] = v32;
            PyObject *g, *ge, *ex;
            if (history(st, &g, &ge, &ex)) {
                Py_XDECREF(g); Py_XDECREF(ge); Py_XDECREF(ex);
                goto done;
            }
            const Py_ssize_t lg = PySequence_Fast_GET_SIZE(g), le = PySequence_Fast_GET_SIZE(ex);
            const Py_ssize_t lge = PySequence_Fast_GET_SIZE(ge);
            const Py_ssize_t m = lg > le ? lg : le;
            c32[3 * n + i] = (int32_t)le;
            c32[4 * n + i] = (int32_t)lg;
            PyObject **G = PySequence_Fast_ITEMS(g), **GE = PySequence_Fast_ITEMS(ge),
                     **EX = PySequence_Fast_ITEMS(ex);
            int bad = 0;
            for (Py_ssize_t j = 0; j < m && !bad; j++) {
                int64_t* row = sl + 4 * (off + j);
                row[0] = row[1] = row[2] = row[3] = 0;
                if (j < lg) {
                    long long a = PyLong_AsLongLong(G[j]);
                    if (a == -1 && PyErr_Occurred()) { bad = 1; break; }
                    row[0] = a;
                    if (j < lge && GE[j] != Py_None) {
                        long long b = PyLong_AsLongLong(GE[j]);
                        if (b == -1 && PyErr_Occurred()) { bad = 1; break; }
                        row[1] = b;
                    }
                }
                if (j < le) {
                    if (attr_i64(EX[j], s_start, &row[2]) || attr_i64(EX[j], s_end, &row[3]))
                        bad = 1;
                }
            }
            Py_DECREF(g); Py_DECREF(ge); Py_DECREF(ex);
            if (bad) goto done;
            off += m;
        }
        result = Py_BuildValue("(nnnn)", (Py_ssize_t)osl, (Py_ssize_t)o32, (Py_ssize_t)oout,
                               (Py_ssize_t)nslot);
    }
done:
    for (i = 0; i < got && i < n; i++) Py_XDECREF(S[i]);
    PyMem_Free(S);
    Py_DECREF(reqs);
    return result;
}

/* dataclasses.replace(req, skipped=skipped) for a validated request
 * (scheduler.py:232-234): a new instance of the same class whose __dict__ is a
 * copy of the original's with `skipped` replaced; classes without a __dict__
 * go through the Python fallback `bump(req, skipped)`. */
static PyObject* bumped(PyObject* req, long skipped, PyObject* bump) {
    /* not a dataclass (replace() raises there) or no __dict__: the fallback */
    PyObject* d = PyObject_HasAttr((PyObject*)Py_TYPE(req), s_dc_fields)
                      ? PyObject_GetAttr(req, s_dict) : NULL;
    if (!d || !PyDict_Check(d)) {
        PyErr_Clear();
        Py_XDECREF(d);
        return PyObject_CallFunction(bump, "Ol", req, skipped);
    }
    PyObject* empty = PyTuple_New(0);
    PyObject* obj = empty ? PyBaseObject_Type.tp_new(Py_TYPE(req), empty, NULL) : NULL;
    Py_XDECREF(empty);
    PyObject* nd = obj ? PyObject_GetAttr(obj, s_dict) : NULL;
    PyObject* sk = nd ? PyLong_FromLong(skipped) : NULL;
    if (!sk || PyDict_Update(nd, d) || PyDict_SetItem(nd, s_skipped, sk)) {
        Py_XDECREF(sk); Py_XDECREF(nd); Py_XDECREF(obj); Py_DECREF(d);
        return NULL;
    }
    Py_DECREF(sk); Py_DECREF(nd); Py_DECREF(d);
    return obj;
}

/* The plan's result objects from the device's one read-back (scheduler.py
 * _place's tail, scheduler.py:223-241):
 *   finish(reqs, states, order_addr, refetch_addr, skipped_addr, n, k,
 *          cloud_addr, bump) -> (edge tuple, deferred tuple, refetch frozenset)
 * order: int32 [n] request indices in plan order; refetch, skipped, cloud
 * (cloud_addr 0: no cloud tier): int32 [n] by request index.  Every task's
 * TaskState.skipped is set to its request's updated counter; the deferred
 * requests (plan order after the first k, the offloaded ones excluded) are
 * bumped copies. */
static PyObject* finish(PyObject* self, PyObject* args) {
    (void)self;
    PyObject *reqs_in, *states, *bump;
    Py_ssize_t oa, ra, sa, ca, n, k;
    if (!PyArg_ParseTuple(args, "OOnnnnnnO", &reqs_in, &states, &oa, &ra, &sa, &n, &k, &ca, &bump))
        return NULL;
    PyObject* reqs = PySequence_Fast(reqs_in, "reqs must be a sequence");
    if (!reqs) return NULL;
    if (PySequence_Fast_GET_SIZE(reqs) != n || k < 0 || k > n) {
        Py_DECREF(reqs);
        PyErr_SetString(PyExc_ValueError, "finish: inconsistent sizes");
        return NULL;
    }
    PyObject** R = PySequence_Fast_ITEMS(reqs);
    const int32_t* order = (const int32_t*)oa;
    const int32_t* refetch = (const int32_t*)ra;
    const int32_t* skipped = (const int32_t*)sa;
    const int32_t* cloud = (const int32_t*)ca;
    Py_ssize_t nd = 0;
    for (Py_ssize_t p = k; p < n; p++) nd += !(cloud && cloud[order[p]]);
    PyObject* edge = PyTuple_New(k);
    PyObject* deferred = PyTuple_New(nd);
    PyObject* ref = PySet_New(NULL);
    PyObject* result = NULL;
    if (!edge || !deferred || !ref) goto done;
    Py_ssize_t q = 0;
    for (Py_ssize_t p = 0; p < n; p++) {
        const int32_t j = order[p];
        if (j < 0 || j >= n) {
            PyErr_SetString(PyExc_ValueError, "finish: order index out of range");
            goto done;
        }
        PyObject* req = R[j];
        PyObject* tid = PyObject_GetAttr(req, s_task_id);
        if (!tid) goto done;
        PyObject* st = PyObject_GetItem(states, tid);
        PyObject* sk = st ? PyLong_FromLong(skipped[j]) : NULL;
        int bad = !sk || PyObject_SetAttr(st, s_skipped, sk);
        Py_XDECREF(sk);
        Py_XDECREF(st);
        if (!bad && refetch[j]) bad = PySet_Add(ref, tid);
        Py_DECREF(tid);
        if (bad) goto done;
        if (p < k) {
            Py_INCREF(req);
            PyTuple_SET_ITEM(edge, p, req);
        } else if (!(cloud && cloud[j])) {
            PyObject* b = bumped(req, skipped[j], bump);
            if (!b) goto done;
            PyTuple_SET_ITEM(deferred, q++, b);
        }
    }
    {
        PyObject* fz = PyFrozenSet_New(ref);
        PyObject* tup = fz ? PyTuple_New(3) : NULL;
        if (!tup) {
            Py_XDECREF(fz);
            goto done;
        }
        PyTuple_SET_ITEM(tup, 0, edge);  /* references moved into the tuple */
        PyTuple_SET_ITEM(tup, 1, deferred);
        PyTuple_SET_ITEM(tup, 2, fz);
        edge = deferred = NULL;
        result = tup;
    }
done:
    Py_XDECREF(edge);
    Py_XDECREF(deferred);
    Py_XDECREF(ref);
    Py_DECREF(reqs);
    return result;
}

static PyMethodDef methods[] = {
    {"pack", pack, METH_VARARGS,
     "pack(reqs, states, rank_of, host_addr, capacity, out_bytes) -> (osl, o32, oout, nsl) | None"},
    {"finish", finish, METH_VARARGS,
     "finish(reqs, states, order_addr, refetch_addr, skipped_addr, n, k, cloud_addr, bump)"
     " -> (edge, deferred, refetch_task_ids)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_kr_pack",
                                    "Native packing of planning objects into the fleet SoA.", -1,
                                    methods};

PyMODINIT_FUNC PyInit__kr_pack(void) {
#define INTERN(v, s) if (!((v) = PyUnicode_InternFromString(s))) return NULL
    INTERN(s_task_id, "task_id");
    INTERN(s_gen_starts, "gen_starts");
    INTERN(s_gen_ends, "gen_ends");
    INTERN(s_exec_intervals, "exec_intervals");
    INTERN(s_t_start, "t_start");
    INTERN(s_issued_at, "issued_at");
    INTERN(s_obs_captured_at, "obs_captured_at");
    INTERN(s_accumulated_generation, "accumulated_generation");
    INTERN(s_last_exec_info, "last_exec_info");
    INTERN(s_remaining_actions, "remaining_actions");
    INTERN(s_skipped, "skipped");
    INTERN(s_start, "start");
    INTERN(s_end, "end");
    INTERN(s_dict, "__dict__");
    INTERN(s_dc_fields, "__dataclass_fields__");
#undef INTERN
    return PyModule_Create(&module);
}
